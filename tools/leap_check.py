"""GPU pipeline vs the compiled reference on C3 / C4 / C5 (quick check while iterating).

  python tools/leap_check.py c3 c5 ...
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

gpu = load_native()
ref = ReconLib(os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so"), "ref")
CASES = {
    "c3": ("bird", 64, 64, 40, 2662, 0x64000000, 4096, 0, 64 * 64 * 12),
    "c3c": ("bird", 64, 64, 40, 2662, 0x64000000, 1024, 1, 64 * 64 * 12),
    "c4": ("redrec", 256, 256, 153, 39322, 0x25600000, 4, 0, 1_500_000),
    "c4c": ("redrec", 256, 256, 153, 39322, 0x25600000, 4, 1, 1_500_000),
    "c5": ("bird", 512, 512, 307, 157286, 0x51200000, 4, 0, 11_000_000),
}
for arg in sys.argv[1:]:
    # name[@first[:count]]
    name, _, rng = arg.partition("@")
    solver, W, H, hp, k, seed, n, preset, ms = CASES[name]
    if rng:
        a, _, b = rng.partition(":")
        seed += int(a, 0)
        n = int(b) if b else n
    occ = sample_grids(seed, n, W, H, k)
    t = time.time()
    g = gpu.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
    tg = time.time() - t
    t = time.time()
    r = ref.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
    tr = time.time() - t
    bad = []
    for key in ("status", "batch_count", "path_count", "total_displacement"):
        if not np.array_equal(g[key], r[key]):
            bad.append(key)
    nmb = 0
    for i in np.nonzero(r["status"] == 0)[0]:
        d = int(r["total_displacement"][i])
        if not np.array_equal(g["move_batch"][i * ms:i * ms + d], r["move_batch"][i * ms:i * ms + d]):
            nmb += 1
    throws = [hex(seed + int(i)) for i in np.nonzero(r["status"] != 0)[0]]
    print(f"{name}: n={n} gpu {tg:.2f}s ref {tr:.2f}s mismatch={bad} move_batch_mismatch={nmb} "
          f"ref_throws={len(throws)} {throws[:25]} nb0={int(r['batch_count'][0])}", flush=True)
