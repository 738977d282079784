"""Reference CPU throughput on THIS host, for every BASELINE config: the
compiled reference (oracle/_ref, built from the reference's own sources) on
bounded samples, std::thread over every host thread (RECON_REF_THREADS), the
same seeded inputs the GPU numbers use.  Prints one JSON line per config.

  python tools/cpu_baselines.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_chains, sample_grids  # noqa: E402

cores = os.cpu_count() or 1
os.environ["RECON_REF_THREADS"] = str(cores)
ref = ReconLib(os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so"), "ref")


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def grid(name, solver, W, H, hp, k, seed, n, single=False):
    occ = sample_grids(seed, n, W, H, k)
    if single:
        os.environ["RECON_REF_THREADS"] = "1"
        dt = min(timed(lambda: ref.grid_solve_batch(solver, occ, 1, W, H, hp, host=True, with_events=False))
                 for _ in range(3))
        os.environ["RECON_REF_THREADS"] = str(cores)
        return {name: {"latency_ms": dt * 1e3, "threads": 1}}
    dt = timed(lambda: ref.grid_solve_batch(solver, occ, n, W, H, hp, host=True, with_events=False))
    return {name: {"grids_per_s": n / dt, "sample": n, "threads": cores}}


def pipeline(name, solver, W, H, hp, k, seed, n, preset):
    occ = sample_grids(seed, n, W, H, k)
    ms = W * H * (W + H)
    dt = timed(lambda: ref.pipeline_batch(solver, occ, n, W, H, hp, preset, ms))
    return {name: {"grids_per_s": n / dt, "sample": n, "threads": cores}}


def chains(name, n, k, tl, th, seed, count):
    occ = sample_chains(seed, count, n, k)
    dt = timed(lambda: ref.solve_1d_batch(occ, count, n, tl, th))
    return {name: {"chains_per_s": count / dt, "sample": count, "threads": cores}}


CASES = [
    lambda: grid("c1_redrec_single", "redrec", 32, 32, 16, 614, 1, 1, single=True),
    lambda: grid("c1_redrec_batch", "redrec", 32, 32, 16, 614, 1, 2048),
    lambda: chains("c2_chains", 1024, 563, 256, 767, 0x1D000000, 16384),
    lambda: grid("c3_bird_solve", "bird", 64, 64, 40, 2662, 0x64000000, 1024),
    lambda: pipeline("c3_bird_batching_none", "bird", 64, 64, 40, 2662, 0x64000000, 512, 0),
    lambda: grid("c4_redrec_h128_single", "redrec", 256, 256, 128, 39322, 256, 1, single=True),
    lambda: grid("c4_redrec_h153_single", "redrec", 256, 256, 153, 39322, 257, 1, single=True),
    lambda: grid("c4_bird_h153_single", "bird", 256, 256, 153, 39322, 257, 1, single=True),
    lambda: grid("r256_redrec_batch", "redrec", 256, 256, 153, 39322, 0x25600000, 64),
    lambda: grid("r256_bird_batch", "bird", 256, 256, 153, 39322, 0x25600000, 64),
    lambda: grid("c5_bird_solve", "bird", 512, 512, 307, 157286, 0x51200000, 16),
]

if __name__ == "__main__":
    print(json.dumps({"host_threads": cores}), flush=True)
    for case in CASES:
        print(json.dumps(case()), flush=True)
