"""Extended randomized parity sweep (one-off, beyond the test suite): batched
grid solves and the solve -> batching pipeline on random shapes, loadings and
band heights, device vs the compiled reference, every instance compared.

  python tools/parity_sweep.py [shapes] [seed]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import LIB_PATH  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so")


def main():
    shapes = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2504)
    gpu, ref = ReconLib(LIB_PATH, "b200"), ReconLib(REF, "ref")
    t0 = time.time()
    bad = 0
    checked = 0
    for it in range(shapes):
        W = int(rng.integers(4, 200))
        H = int(rng.integers(4, 200))
        hp = int(rng.integers(1, H))
        fill = float(rng.uniform(0.5, 0.8))
        k = min(W * H, max(W * hp, int(fill * W * H)))
        n = int(rng.integers(1, 96))
        seed = int(rng.integers(0, 1 << 30))
        occ = sample_grids(seed, n, W, H, k)
        for solver in ("redrec", "bird"):
            g = gpu.grid_solve_batch(solver, occ, n, W, H, hp)
            r = ref.grid_solve_batch(solver, occ, n, W, H, hp)
            ok = all(np.array_equal(g[key], r[key]) for key in ("path_count", "total_displacement", "status"))
            S = W * hp
            for i in range(n):
                P = int(r["path_count"][i])
                for key in ("path_src", "path_dst"):
                    ok = ok and np.array_equal(g[key][i * S:i * S + P], r[key][i * S:i * S + P])
            preset = int(rng.integers(0, 2))
            ms = W * H * 16
            gp = gpu.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
            rp = ref.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
            for key in ("status", "batch_count", "path_count", "total_displacement"):
                ok = ok and np.array_equal(gp[key], rp[key])
            for i in np.nonzero(rp["status"] == 0)[0]:
                d = int(rp["total_displacement"][i])
                ok = ok and np.array_equal(gp["move_batch"][i * ms:i * ms + d], rp["move_batch"][i * ms:i * ms + d])
            checked += 2 * n
            if not ok:
                bad += 1
                print("MISMATCH", dict(W=W, H=H, hp=hp, k=k, n=n, seed=seed, solver=solver, preset=preset), flush=True)
    print({"shapes": shapes, "instances_checked": checked, "mismatching_shapes": bad, "s": round(time.time() - t0, 1)})
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
