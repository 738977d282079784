"""Earliest batch where the device schedule differs from the compiled
reference (debugging aid): python tools/first_diff.py c5|c4 [index]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

CASES = {
    "c4": ("redrec", 256, 256, 153, 39322, 0x25600000, 1_500_000),
    "c5": ("bird", 512, 512, 307, 157286, 0x51200000, 12_000_000),
}
name = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
solver, W, H, hp, k, seed, ms = CASES[name]
occ = sample_grids(seed + idx, 1, W, H, k)
g = load_native().pipeline_batch(solver, occ, 1, W, H, hp, 0, ms)
r = ReconLib(os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so"), "ref").pipeline_batch(solver, occ, 1, W, H, hp, 0, ms)
P = int(r["path_count"][0])
src, dst = r["path_src"][:P], r["path_dst"][:P]
ln = np.abs(dst // H - src // H) + np.abs(dst % H - src % H)
base = np.concatenate([[0], np.cumsum(ln)])
D = int(base[-1])
mg, mr = g["move_batch"][:D].astype(np.int64), r["move_batch"][:D].astype(np.int64)
print("status", g["status"][0], r["status"][0], "nb", g["batch_count"][0], r["batch_count"][0])
bad = np.nonzero(mg != mr)[0]
if len(bad) == 0:
    print("schedules equal")
    sys.exit(0)
b0 = int(min(mg[bad].min(), mr[bad].min()))
pid_of = np.repeat(np.arange(P), ln)
kk = np.arange(D) - base[pid_of]
print("first differing batch", b0, "#differing moves", len(bad))
for lab, m in (("gpu", mg), ("ref", mr)):
    sel = np.nonzero(m == b0)[0]
    print(lab, "moves at", b0, ":", len(sel))
    for s in sel:
        if mg[s] != mr[s]:
            p = pid_of[s]
            print(f"   pid {p} k {kk[s]} len {ln[p]} gpu {mg[s]} ref {mr[s]} src {src[p] // H},{src[p] % H} dst {dst[p] // H},{dst[p] % H}")
# paths whose first move differs
for p in np.unique(pid_of[bad])[:10]:
    sl = slice(base[p], base[p + 1])
    print("pid", p, "gpu", mg[sl][:6], "ref", mr[sl][:6])
