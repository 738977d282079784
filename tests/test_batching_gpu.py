"""GPU parity of batch_moves (recon_batch_moves) and of the fused
solve -> occupancy DAG -> batching pipeline (recon_pipeline_batch_run)."""
import numpy as np
import pytest

from helpers import random_band_instance
from paper_2504_06182_b200.abi import InputError
from paper_2504_06182_b200.inputs import grid_from_vertices, sample_grids

pytestmark = pytest.mark.gpu


def _cmp_pipeline(a, b, stride_moves):
    assert np.array_equal(a["status"], b["status"])
    assert np.array_equal(a["detail"], b["detail"])
    assert np.array_equal(a["batch_count"], b["batch_count"])
    assert np.array_equal(a["path_count"], b["path_count"])
    assert np.array_equal(a["total_displacement"], b["total_displacement"])
    for i in np.nonzero(a["status"] == 0)[0]:
        d = int(a["total_displacement"][i])
        mb_a = a["move_batch"][i * stride_moves:i * stride_moves + d]
        mb_b = b["move_batch"][i * stride_moves:i * stride_moves + d]
        assert np.array_equal(mb_a, mb_b), i


@pytest.mark.parametrize("solver", ["redrec", "bird"])
@pytest.mark.parametrize("preset", [0, 1])
def test_pipeline_random_matches_oracle(gpu, oracle, solver, preset):
    rng = np.random.default_rng(0xba7c + preset)
    for it in range(60):
        occ, W, H, hp = random_band_instance(rng, 20, 30, critical=bool(it % 2))
        ms = W * H * (W + H)
        g = gpu.pipeline_batch(solver, occ, 1, W, H, hp, preset, ms)
        o = oracle.pipeline_batch(solver, occ, 1, W, H, hp, preset, ms)
        _cmp_pipeline(g, o, ms)


@pytest.mark.parametrize("preset", [0, 1])
def test_pipeline_c3_bird_matches_reference(gpu, ref, preset):
    # C3: 64x64, h'=40, 2662 atoms; seed 0x6400001d throws "no progress" with preset none
    W = H = 64
    n = 48
    occ = sample_grids(0x64000000, n, W, H, 2662)
    ms = 64 * 64 * 12
    g = gpu.pipeline_batch("bird", occ, n, W, H, 40, preset, ms)
    r = ref.pipeline_batch("bird", occ, n, W, H, 40, preset, ms)
    _cmp_pipeline(g, r, ms)
    if preset == 0:
        assert g["status"][0x1d] == 1  # InputError, batching.cpp:127-128


def _problem(W, H, S):
    return grid_from_vertices(S, W, H)


def test_batch_moves_reference_cases(gpu):
    # test_batching.cpp:59-155 pinned batch counts
    occ = _problem(6, 1, [0, 3])
    for preset in (0, 1):
        mb, nb = gpu.batch_moves(6, 1, occ, [[0, 1], [3, 4]], [], preset)
        assert nb == 1
    mb, nb = gpu.batch_moves(4, 1, _problem(4, 1, [0]), [[0, 1, 2, 3]], [])
    assert nb == 3
    H = 3
    gid = lambda x, y: x * H + y  # noqa: E731
    occ = _problem(3, 3, [gid(0, 0), gid(2, 0)])
    paths = [[gid(0, 0), gid(0, 1)], [gid(2, 0), gid(2, 1)]]
    assert gpu.batch_moves(3, 3, occ, paths, [], 0)[1] == 1
    assert gpu.batch_moves(3, 3, occ, paths, [], 1)[1] == 2
    occ = _problem(5, 1, [1, 2])
    mb, nb = gpu.batch_moves(5, 1, occ, [[2, 3], [1, 2]], [[0, 1]])
    assert nb == 2 and mb.tolist() == [0, 1]
    mb, nb = gpu.batch_moves(5, 1, occ, [[2, 3], [1, 2]], [])
    assert nb == 2
    mb, nb = gpu.batch_moves(3, 1, _problem(3, 1, [1]), [[1]], [])
    assert nb == 0
    # edge-level release (test_batching.cpp:137-155)
    H = 4
    gid = lambda x, y: x * H + y  # noqa: E731
    a0, a1, a2, a3, b0 = gid(0, 0), gid(0, 1), gid(0, 2), gid(0, 3), gid(1, 0)
    occ = _problem(2, 4, [a0, b0])
    paths = [[a0, a1, a2, a3], [b0, a0]]
    assert gpu.batch_moves(2, 4, occ, paths, [[0, 1]])[1] == 4
    assert gpu.batch_moves(2, 4, occ, paths, [[0, 1]], edge_level=True)[1] == 3
    # cyclic dag throws (test_batching.cpp:157-172)
    with pytest.raises(InputError):
        gpu.batch_moves(6, 1, _problem(6, 1, [0, 3]), [[0, 1], [3, 4]], [[0, 1], [1, 0]])


def test_batch_moves_random_matches_reference(gpu, ref):
    """Explicit-path entry point on solver outputs, both presets, edge-level too."""
    rng = np.random.default_rng(0xfeed)
    from paper_2504_06182_b200.abi import ReconError
    for it in range(40):
        occ, W, H, hp = random_band_instance(rng, 12, 16, critical=bool(it % 2))
        sol = ref.grid_solve("bird" if it % 3 else "redrec", occ, W, H, hp, with_dag=True)
        paths = []
        for s, t in zip(sol.path_src, sol.path_dst):
            xs, ys, xt, yt = s // H, s % H, t // H, t % H
            v = [s]
            x, y = xs, ys
            while x != xt:
                x += 1 if xt > x else -1
                v.append(x * H + y)
            while y != yt:
                y += 1 if yt > y else -1
                v.append(x * H + y)
            paths.append(v)
        for preset in (0, 1):
            for el in (False, True):
                try:
                    r = ref.batch_moves(W, H, occ, paths, sol.dag, preset, el)
                    er = None
                except ReconError as e:
                    r, er = None, type(e).__name__
                try:
                    g = gpu.batch_moves(W, H, occ, paths, sol.dag, preset, el)
                    eg = None
                except ReconError as e:
                    g, eg = None, type(e).__name__
                assert er == eg
                if r is not None:
                    assert r[1] == g[1] and np.array_equal(r[0], g[0]), (it, preset, el)


@pytest.mark.parametrize("solver,W,hp,k,n", [("bird", 64, 40, 2662, 700), ("redrec", 32, 16, 614, 1200)])
@pytest.mark.parametrize("preset", [0, 1])
def test_pipeline_many_instances_matches_reference(gpu, ref, solver, W, hp, k, n, preset):
    """Batches of >= 4 instances per SM take the many-instance pipeline: the
    shared-memory DAG build, the move log + scatter, blocker counts in shared
    memory and the record ready list."""
    occ = sample_grids(0x64100000 + W, n, W, W, k)
    ms = W * W * 12
    g = gpu.pipeline_batch(solver, occ, n, W, W, hp, preset, ms)
    r = ref.pipeline_batch(solver, occ, n, W, W, hp, preset, ms)
    _cmp_pipeline(g, r, ms)
    assert (g["status"] == 0).sum() > n // 2


def test_pipeline_failed_instances_report_detail(gpu, ref):
    """the host pipeline returns each failed instance's detail —
    InfeasibleError from the solve (problem.hpp:115) and the batching
    no-progress InputError (batching.cpp:127-128) — next to solved ones."""
    W = H = 64
    occ = np.concatenate([sample_grids(0x64000000, 30, W, H, 2662), sample_grids(7, 1, W, H, 2000),
                          sample_grids(0x6400001d, 1, W, H, 2662)])
    ms = W * H * 12
    g = gpu.pipeline_batch("bird", occ, 32, W, H, 40, 0, ms)
    r = ref.pipeline_batch("bird", occ, 32, W, H, 40, 0, ms)
    _cmp_pipeline(g, r, ms)
    assert g["status"][30] == 2 and g["detail"][30] != 0  # InfeasibleError
    assert g["status"][31] == 1 and g["detail"][31] != 0  # no progress
    assert (g["detail"][g["status"] == 0] == 0).all()
