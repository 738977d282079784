"""Times the general batch_moves entry point (recon_batch_moves: explicit
vertex paths + a given dag, what the C++ shim's batch_moves calls) on solver
output, against the fused pipeline on the same instance.

  python tools/probe_explicit.py [W H h' atoms seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_06182_b200 import LIB_PATH  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402


def staircase(H, s, t):
    xs, ys, xt, yt = s // H, s % H, t // H, t % H
    dx, dy = (1 if xt > xs else -1), (1 if yt > ys else -1)
    v = [x * H + ys for x in range(xs, xt + dx, dx)] if xs != xt else [s]
    if ys != yt:
        v += [xt * H + y for y in range(ys + dy, yt + dy, dy)]
    return v


def main():
    W, H, hp, k, seed = [int(x, 0) for x in sys.argv[1:6]] if len(sys.argv) > 5 else (256, 256, 153, 39322, 257)
    lib = ReconLib(LIB_PATH, "b200")
    occ = sample_grids(seed, 1, W, H, k)
    ms = W * H * 48
    t0 = time.perf_counter()
    pipe = lib.pipeline_batch("redrec", occ, 1, W, H, hp, 0, ms)
    t_pipe = time.perf_counter() - t0
    P = int(pipe["path_count"][0])
    src, dst = pipe["path_src"][:P], pipe["path_dst"][:P]
    paths = [staircase(H, int(s), int(t)) for s, t in zip(src, dst)]
    edges = lib.occupancy_dag(W, H, src, dst)
    for rep in range(2):
        t0 = time.perf_counter()
        mb, nb = lib.batch_moves(W, H, occ, paths, edges, 0)
        t_exp = time.perf_counter() - t0
    D = int(pipe["total_displacement"][0])
    assert int(pipe["status"][0]) == 0, ("pipeline status", int(pipe["status"][0]))
    same = nb == int(pipe["batch_count"][0]) and np.array_equal(mb, pipe["move_batch"][:D])
    print({"W": W, "H": H, "paths": P, "moves": D, "edges": len(edges), "batches": nb,
           "explicit_batch_moves_s": round(t_exp, 4), "pipeline_s (solve+dag+batch, host)": round(t_pipe, 4),
           "same_schedule": bool(same)})


if __name__ == "__main__":
    main()
