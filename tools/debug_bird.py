"""Finds the first bird instance where the GPU differs from the oracle and dumps per-event stats."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import random_band_instance  # noqa: E402
from paper_2504_06182_b200 import LIB_PATH, load_native  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402

gpu = load_native()
orc = ReconLib(os.path.join(ROOT, "oracle", "librecon_oracle.so"))
raw = C.CDLL(LIB_PATH)
rng = np.random.default_rng(0x5ed5ec)
for it in range(400):
    occ, W, H, hp = random_band_instance(rng, 16, 24, critical=bool(it % 2))
    try:
        g = gpu.grid_solve("bird", occ, W, H, hp)
        o = orc.grid_solve("bird", occ, W, H, hp)
    except Exception as e:
        continue
    if np.array_equal(g.path_src, o.path_src) and np.array_equal(g.path_dst, o.path_dst):
        continue
    print("mismatch it", it, "W H hp", W, H, hp, "paths", len(g.path_src), len(o.path_src))
    out = np.zeros(8 + 8 * W, np.int64)
    raw.recon_debug_grid_phases(1, occ.ctypes.data_as(C.c_void_p), W, H, hp, out.ctypes.data_as(C.c_void_p), len(out))
    ev = out[8:].reshape(W, 8)
    print("events order", list(g.events), list(o.events))
    for e in range(W):
        ge = [(s, d) for s, d, v in zip(g.path_src, g.path_dst, g.path_event) if v == e]
        oe = [(s, d) for s, d, v in zip(o.path_src, o.path_dst, o.path_event) if v == e]
        if ge != oe:
            n1 = sum(1 for x in g.events if True)  # placeholder
            print("first differing event", e, "column", g.events[e])
            print(" gpu  ", ge)
            print(" orc  ", oe)
            print(" dbg rows (holes, lev_t, lev_b, found_t, found_b, a, b):")
            for r in ev:
                if r[0] or r[5] or r[6]:
                    print("   ", list(r[:7]))
            break
    wpc = (H + 63) // 64
    grid = [[(int(occ[x * wpc + y // 64]) >> (y % 64)) & 1 for y in range(H)] for x in range(W)]
    for y in range(H - 1, -1, -1):
        print("".join("#" if grid[x][y] else "." for x in range(W)), H - 1 - y)
    break
