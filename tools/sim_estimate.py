"""estimate_success (SPEC.md sim) on the device: success probability with its
binomial standard error and per-trial operation counts, for the paper's
32x64 grid with a 32x32 target (§V-C), both solvers, batching off
and on.  Model parameters are the SPEC defaults (durations are calibration
knobs, not paper constants).

  python tools/sim_estimate.py [trials] [tau_seconds]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
lib = load_native()
W, H, hp = 32, 64, 32
occ = sample_grids(0x5EED0000, n, W, H, round(0.6 * W * H))
for solver in ("redrec", "bird"):
    for batching in (False, True):
        t0 = time.perf_counter()
        r = lib.sim_run(occ, n, W, H, hp, 0x5EED0000, solver=solver, batching=batching, max_cycles=50,
                        p_nu=0.985, p_alpha=0.985, tau=tau)
        dt = time.perf_counter() - t0
        p = float(r["success"].mean())
        print(json.dumps({"solver": solver, "batching": batching, "trials": n, "tau_s": tau, "p_bar": p,
                          "stderr": (p * (1 - p) / n) ** 0.5, "cycles_mean": float(r["cycles"].mean()),
                          "N_nu_mean": float(r["n_nu"].mean()), "N_alpha_mean": float(r["n_alpha"].mean()),
                          "NB_nu_mean": float(r["nb_nu"].mean()), "NB_alpha_mean": float(r["nb_alpha"].mean()),
                          "elapsed_model_s_mean": float(r["elapsed"].mean()), "wall_s": round(dt, 3)}), flush=True)
