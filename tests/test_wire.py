"""Wire formats: recon_solution_json / recon_batch_schedule_json produce the
reference's solution_to_json / batch_schedule_to_json text (io.cpp:81-164).

The reference prints through nlohmann::ordered_json::dump(2); its vendored
json.hpp is not in the reference tree, so the layout is pinned against the
stock library's, which Python's json.dumps(indent=2) reproduces for these
documents (one value per line, two-space indent, "[]" for empty arrays,
", " never used).  The content (schedule order, dag, paths, batch order and
tags) comes from the compiled reference (oracle/_ref) building its own
Solution / BatchSchedule objects.
"""
import json

import numpy as np
import pytest

from validate_cases import pipeline_instances


def one_bend(H, s, t):
    xs, ys, xt, yt = s // H, s % H, t // H, t % H
    v = [(xs, ys)]
    x, y = xs, ys
    while x != xt:
        x += 1 if xt > x else -1
        v.append((x, y))
    while y != yt:
        y += 1 if yt > y else -1
        v.append((x, y))
    return v


def expected_solution(H, src, dst, order, dag, displaced, total):
    paths = [one_bend(H, int(s), int(t)) for s, t in zip(src, dst)]
    order = range(len(paths)) if order is None else order
    moves = [[list(paths[q][k]), list(paths[q][k + 1])] for q in order for k in range(len(paths[q]) - 1)]
    obj = {"moves": moves, "dag_edges": [[int(a), int(b)] for a, b in dag],
           "paths": [[list(v) for v in p] for p in paths],
           "stats": {"displaced_tokens": int(displaced), "total_displacement": int(total)}}
    return (json.dumps(obj, indent=2) + "\n").encode()


def expected_batches(H, src, dst, mb, nb, preset):
    paths = [one_bend(H, int(s), int(t)) for s, t in zip(src, dst)]
    batches = [[] for _ in range(nb)]
    m = 0
    for p in paths:
        for k in range(len(p) - 1):
            batches[mb[m]].append((p[k], p[k + 1]))
            m += 1
    out = []
    for b in batches:
        if not b:
            continue
        ax = dr = None
        if preset == 1:
            (fx, fy), (tx, ty) = b[0]
            ax, dr = ("col", "up") if ty > fy else ("col", "down") if ty < fy else ("row", "left") if tx < fx else ("row", "right")
        out.append({"axis": ax, "dir": dr, "moves": [[list(f), list(t)] for f, t in b]})
    return (json.dumps({"batches": out}, indent=2) + "\n").encode()


CFGS = [("redrec", 32, 32, 16, 614, 1, 3, 0), ("bird", 24, 20, 9, 260, 77, 3, 1), ("redrec", 16, 24, 11, 240, 5, 2, 1)]


@pytest.fixture(scope="module")
def cases(ref):
    out = []
    for cfg in CFGS:
        for c in pipeline_instances(ref, *cfg):
            c["dag"] = ref.occupancy_dag(c["width"], c["height"], c["path_src"], c["path_dst"])
            out.append(c)
    return out


def _check(lib, c, rng):
    W, H = c["width"], c["height"]
    src, dst = c["path_src"], c["path_dst"]
    P = len(src)
    for order in (None, rng.permutation(P).astype(np.int32)):
        got = lib.solution_json(W, H, src, dst, order, c["dag"], P, int(c["total_displacement"][0]))
        assert got == expected_solution(H, src, dst, order, c["dag"], P, int(c["total_displacement"][0]))
    got = lib.batch_schedule_json(W, H, src, dst, c["move_batch"], int(c["batch_count"][0]), c["preset"])
    assert got == expected_batches(H, src, dst, c["move_batch"], int(c["batch_count"][0]), c["preset"])


def test_checkers_match_layout(ref, oracle, cases):
    rng = np.random.default_rng(7)
    for c in cases:
        _check(ref, c, rng)
        _check(oracle, c, rng)
    # empty documents
    for lib in (ref, oracle):
        assert lib.solution_json(4, 4, [], []) == expected_solution(4, [], [], None, [], 0, 0)
        assert lib.batch_schedule_json(4, 4, [], [], [], 0) == b'{\n  "batches": []\n}\n'


@pytest.mark.gpu
def test_device_json_matches(gpu, cases):
    rng = np.random.default_rng(7)
    for c in cases:
        _check(gpu, c, rng)
    assert gpu.solution_json(4, 4, [], []) == expected_solution(4, [], [], None, [], 0, 0)
    assert gpu.batch_schedule_json(4, 4, [], [], [], 0) == b'{\n  "batches": []\n}\n'


@pytest.mark.gpu
def test_device_json_c4_scale(gpu, oracle):
    """One C4 red-rec pipeline instance (256x256, ~1M moves): the device text
    equals the oracle's byte for byte (tens of MB)."""
    c = pipeline_instances(gpu, "redrec", 256, 256, 153, 39322, 257, 1, 0)[0]
    dag = gpu.occupancy_dag(256, 256, c["path_src"], c["path_dst"])
    args = (256, 256, c["path_src"], c["path_dst"], None, dag, len(c["path_src"]), int(c["total_displacement"][0]))
    a, b = gpu.solution_json(*args), oracle.solution_json(*args)
    assert len(a) > 10_000_000 and a == b
    bargs = (256, 256, c["path_src"], c["path_dst"], c["move_batch"], int(c["batch_count"][0]), 0)
    assert gpu.batch_schedule_json(*bargs) == oracle.batch_schedule_json(*bargs)
