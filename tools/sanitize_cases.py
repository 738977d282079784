"""Small invocations of every kernel family, for compute-sanitizer
(tools/sanitize.sh): red-rec / bird solves (batched + lone-instance shapes),
band and general 1D chains, the occupancy DAG, the fused pipeline (leap +
wide + warp batching, both presets, the many-instance batch-by-batch
variants), the stats record, the validators, the JSON writers and the loss
simulation.  Each result is also checked against the oracle, so a run that
exits 0 under the sanitizer computed the right answer.

  python tools/sanitize_cases.py [family ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_chains, sample_grids  # noqa: E402

gpu = load_native()
oracle = ReconLib(os.path.join(ROOT, "oracle", "librecon_oracle.so"), "oracle")


def same(a, b, keys):
    for k in keys:
        assert np.array_equal(a[k], b[k]), k


def solves():
    for W, H, hp, k, n in ((32, 32, 16, 614, 8), (64, 64, 40, 2662, 4), (128, 128, 77, 10000, 1)):
        occ = sample_grids(0x5A000000 + W, n, W, H, k)
        for solver in ("redrec", "bird"):
            g = gpu.grid_solve_batch(solver, occ, n, W, H, hp, host=True, with_events=False)
            o = oracle.grid_solve_batch(solver, occ, n, W, H, hp, host=True, with_events=False)
            same(g, o, ("path_count", "total_displacement", "status"))
            for i in range(n):  # the used slots of every instance
                P, s0 = int(o["path_count"][i]), i * W * hp
                assert np.array_equal(g["path_src"][s0:s0 + P], o["path_src"][s0:s0 + P])
                assert np.array_equal(g["path_dst"][s0:s0 + P], o["path_dst"][s0:s0 + P])
            one = gpu.grid_solve(solver, occ[: W * ((H + 63) // 64)], W, H, hp, with_dag=True)
            ref1 = oracle.grid_solve(solver, occ[: W * ((H + 63) // 64)], W, H, hp, with_dag=True)
            assert np.array_equal(one.dag, ref1.dag)


def chains():
    occ = sample_chains(0x1D000000, 64, 1024, 563)
    g = gpu.solve_1d_batch(occ, 64, 1024, 256, 767)
    o = oracle.solve_1d_batch(occ, 64, 1024, 256, 767)
    for key in g:
        assert np.array_equal(g[key], o[key]), key
    rng = np.random.default_rng(7)
    for _ in range(4):
        n = 200
        S = np.sort(rng.choice(n, 90, replace=False))
        T = np.sort(rng.choice(n, 60, replace=False))
        a = gpu.solve_1d(n, S, T)
        b = oracle.solve_1d(n, S, T)
        assert np.array_equal(a.path_src, b.path_src) and np.array_equal(a.dag, b.dag)


def pipeline():
    from digest import pipeline_digests
    for solver, W, H, hp, k, n, preset in (("bird", 64, 64, 40, 2662, 24, 0), ("bird", 64, 64, 40, 2662, 8, 1),
                                           ("redrec", 48, 48, 29, 1383, 6, 0), ("redrec", 48, 48, 29, 1383, 4, 1)):
        occ = sample_grids(0x64000000, n, W, H, k)
        ms = W * H * 12
        g = gpu.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
        o = oracle.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
        assert np.array_equal(g["status"], o["status"]) and np.array_equal(g["batch_count"], o["batch_count"])
        assert np.array_equal(pipeline_digests(g, n, W * hp, ms), pipeline_digests(o, n, W * hp, ms))


def stats():
    from paper_2504_06182_b200.pipeline import C3, PipelineRunner
    r = PipelineRunner(gpu, C3, 16)
    occ = sample_grids(C3.seed_base, 16, 64, 64, C3.atoms)
    r.load(occ, 16)
    r.run(16)
    st = r.stats(16)
    o = oracle.pipeline_batch("bird", occ, 16, 64, 64, 40, 0, C3.move_stride)
    assert np.array_equal(st, oracle.pipeline_stats_host(o, 16, 64, 40, C3.move_stride))


def validators():
    from validate_cases import DAG_OCCUPANCY, pipeline_instances, run, with_dag
    for base in pipeline_instances(oracle, "bird", 32, 32, 16, 614, 1, 2, 0):
        c = with_dag(base, DAG_OCCUPANCY)
        assert run(gpu, c) == run(oracle, c)


def wire():
    occ = sample_grids(1, 1, 32, 32, 614)
    o = oracle.pipeline_batch("bird", occ, 1, 32, 32, 16, 0, 32 * 32 * 12)
    P, D = int(o["path_count"][0]), int(o["total_displacement"][0])
    src, dst = o["path_src"][:P], o["path_dst"][:P]
    assert gpu.solution_json(32, 32, src, dst, displaced=P, total=D) == oracle.solution_json(
        32, 32, src, dst, displaced=P, total=D)
    mb = o["move_batch"][:D]
    nb = int(o["batch_count"][0])
    assert gpu.batch_schedule_json(32, 32, src, dst, mb, nb) == oracle.batch_schedule_json(32, 32, src, dst, mb, nb)


def sim():
    occ = sample_grids(0x51A00000, 8, 32, 32, 614)
    for batching in (False, True):
        g = gpu.sim_run(occ, 8, 32, 32, 16, 0x1234, solver="bird", batching=batching, max_cycles=4)
        o = oracle.sim_run(occ, 8, 32, 32, 16, 0x1234, solver="bird", batching=batching, max_cycles=4)
        for key in g:
            assert np.array_equal(g[key], o[key]), key


FAMILIES = {"solves": solves, "chains": chains, "pipeline": pipeline, "stats": stats, "validators": validators,
            "wire": wire, "sim": sim}

if __name__ == "__main__":
    names = sys.argv[1:] or list(FAMILIES)
    for name in names:
        FAMILIES[name]()
        print(f"{name}: ok", flush=True)
