"""Checks a ReconLib against the committed golden fixtures (tests/golden/*.npz,
generated from the compiled reference by tests/golden/make_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SOLVER = {"c1_redrec": "redrec", "c1_bird": "bird", "c3_bird": "bird", "c3_redrec_coldir": "redrec",
          "g128_redrec": "redrec", "c3_bird_throw": "bird"}


def grid_fixtures():
    return sorted(n for n in SOLVER if os.path.exists(os.path.join(GOLDEN, n + ".npz")))


def check_grid_fixture(lib, name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    W, H, hp, k, _, count = (int(x) for x in d["shape"])
    wpc = (H + 63) // 64
    solver = SOLVER[name]
    po = do = 0
    for i in range(count):
        r = lib.grid_solve(solver, d["occ"][i * W * wpc:(i + 1) * W * wpc], W, H, hp, with_dag=True)
        pc, dc = int(d["path_count"][i]), int(d["dag_count"][i])
        assert np.array_equal(r.path_src, d["path_src"][po:po + pc]), (name, i)
        assert np.array_equal(r.path_dst, d["path_dst"][po:po + pc]), (name, i)
        assert np.array_equal(r.path_event, d["path_event"][po:po + pc]), (name, i)
        assert np.array_equal(r.dag, d["dag"][do:do + dc]), (name, i)
        assert r.total_displacement == int(d["total_displacement"][i])
        per = 4 if solver == "redrec" else 1
        assert np.array_equal(r.events, d["events"][i * W * per:(i + 1) * W * per])
        po += pc
        do += dc
    if "preset" in d:
        ms = W * H * 12
        pb = lib.pipeline_batch(solver, d["occ"], count, W, H, hp, int(d["preset"][0]), ms)
        assert np.array_equal(pb["status"], d["batch_status"])
        assert np.array_equal(pb["batch_count"], d["batch_count"])
        mo = 0
        for i in range(count):
            disp = int(d["total_displacement"][i])
            if d["batch_status"][i] == 0:
                assert np.array_equal(pb["move_batch"][i * ms:i * ms + disp], d["move_batch"][mo:mo + disp])
            mo += disp


def check_chain_fixture(lib):
    d = np.load(os.path.join(GOLDEN, "c2_chains.npz"))
    n, k, tl, th, _, count = (int(x) for x in d["shape"])
    r = lib.solve_1d_batch(d["occ"], count, n, tl, th)
    for key in ("path_src", "path_dst", "total_displacement", "displaced", "status"):
        assert np.array_equal(r[key], d[key]), key
