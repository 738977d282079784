"""Phase cycle breakdown of the pipeline batching warp (library built with
RECON_NVCC_EXTRA=-DRECON_BATCH_PROF).

  python tools/batch_prof.py c5 [count]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

CASES = {
    "c3": ("bird", 64, 64, 40, 2662, 0x64000000, 0, 64 * 64 * 12),
    "c4": ("redrec", 256, 256, 153, 39322, 0x25600000, 0, 1_500_000),
    "c5": ("bird", 512, 512, 307, 157286, 0x51200000, 0, 12_000_000),
}
gpu = load_native()
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
solver, W, H, hp, k, seed, preset, ms = CASES[name]
occ = sample_grids(seed, n, W, H, k)
buf = (C.c_ulonglong * 16)()
wbuf = (C.c_ulonglong * 8)()
vbuf = (C.c_ulonglong * 20)()
gpu.lib.recon_debug_batch_prof(buf, 1)
gpu.lib.recon_debug_wide_prof(wbuf, 1)
gpu.lib.recon_debug_window_prof(vbuf, 1)
t = time.time()
g = gpu.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
dt = time.time() - t
gpu.lib.recon_debug_batch_prof(buf, 1)
gpu.lib.recon_debug_wide_prof(wbuf, 1)
gpu.lib.recon_debug_window_prof(vbuf, 1)
v = list(buf)
vv = list(vbuf)
wv = list(wbuf)
names = ["leap_delta", "leap_apply", "literal", "finish", "general", "n_leap", "n_literal", "n_general", "n_finish",
         "total"]
out = {names[i]: v[i] for i in range(10)}
cyc = {k2: out[k2] / n for k2 in names[:5] + ["total"]}
print(name, n, f"wall {dt:.2f}s", "per-instance Mcycles:", {k2: round(c / 1e6, 2) for k2, c in cyc.items()})
print("counts per instance:", {k2: out[k2] / n for k2 in names[5:9]})
for a, b in (("leap_delta", "n_leap"), ("literal", "n_literal"), ("general", "n_general"), ("finish", "n_finish")):
    if out[b]:
        print(f"  {a}: {out[a] / max(1, out[b] if a != 'leap_delta' else out['n_leap'] + out['n_literal']):.0f} cycles per")
if v[12]:
    print(f"  finish detail: successor loads {v[10] / v[12]:.0f}, decrements+records+lanes {v[11] / v[12]:.0f} cycles per finish")
if v[15]:
    print(f"  leap_delta recomputed in full: {v[15] / n:.0f} per instance (the rest from the cached pair meetings)")
if v[14]:
    print(f"  early finishes: {v[14] / n:.0f} per instance, release_fill {v[13] / v[14]:.0f} cycles")
if wv[4]:
    nbw = wv[3]
    print(f"wide: {wv[4]} instances, {nbw / wv[4]:.0f} batches each; cycles per batch: "
          f"candidates {wv[0] / nbw:.0f}, apply {wv[1] / nbw:.0f}, release {wv[2] / nbw:.0f}")
if vv[7]:
    ni, nbw = vv[7], max(1, vv[4])
    print(f"window: {ni} instances; per instance: {vv[0] / ni:.0f} windows ({vv[1] / ni:.1f} stalled, "
          f"{vv[2] / ni:.1f} overflowed), {vv[3] / ni:.1f} literal batches, {vv[4] / ni:.0f} batches; "
          f"cycles per batch: plan {vv[5] / nbw:.0f}, replay {vv[6] / nbw:.0f}, commit {vv[11] / nbw:.0f}, "
          f"literal+other {vv[10] / nbw:.0f}; finishers per window {vv[8] / max(1, vv[0]):.0f}, "
          f"rounds per window {vv[9] / max(1, vv[0] + vv[2]):.2f}")
    if vv[19]:
        print(f"  pass1 first piece (thread 0): ranges {vv[17] / vv[19]:.0f}, piece {vv[18] / vv[19]:.0f} cycles")
    print(f"  plan per window: scan {vv[12] / max(1, vv[0]):.0f}, pass1 {vv[13] / max(1, vv[0]):.0f}, "
          f"(ranges {vv[16] / max(1, vv[0]):.0f}), pass2 {vv[14] / max(1, vv[0]):.0f}, pass3 {vv[15] / max(1, vv[0]):.0f}, rest {vv[5] / max(1, vv[0]):.0f} cycles")
print("batch_count", g["batch_count"][:4], "status", np.unique(g["status"]))
