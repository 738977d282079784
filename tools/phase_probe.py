"""clock64 phase split of one red-rec solve (plan / phase-1 + pairing loop / phase 3)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import LIB_PATH  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

lib = C.CDLL(LIB_PATH)
for (W, H, hp, k, seed) in [(256, 256, 128, 39322, 256), (256, 256, 153, 39322, 257), (32, 32, 16, 614, 1),
                            (512, 512, 307, 157286, 0x51200000)]:
    occ = sample_grids(seed, 1, W, H, k)
    out = np.zeros(6, np.int64)
    for rep in range(2):
        st = lib.recon_debug_grid_phases(0, occ.ctypes.data_as(C.c_void_p), W, H, hp, out.ctypes.data_as(C.c_void_p), 6)
    c = out
    print(f"{W}x{H} h'={hp}: plan {(c[1]-c[0])/1965:.1f} us, phase1+loop {(c[2]-c[1])/1965:.1f} us, "
          f"phase3 {(c[3]-c[2])/1965:.1f} us (n1={c[4]}, loop events={c[5]//1000}, levels={c[5]%1000}) st={st}")

# bird row pass: per pooled event (holes, levels scanned top/bottom, tokens found, a, b)
for (W, H, hp, k, seed) in [(256, 256, 153, 39322, 257), (512, 512, 307, 157286, 0x51200000), (64, 64, 40, 2662, 0x64000000)]:
    occ = sample_grids(seed, 1, W, H, k)
    out = np.zeros(8 + 8 * W, np.int64)
    lib.recon_debug_grid_phases(1, occ.ctypes.data_as(C.c_void_p), W, H, hp, out.ctypes.data_as(C.c_void_p), len(out))
    ev = out[8:].reshape(W, 8)
    ev = ev[ev[:, 0] > 0]
    print(f"bird {W}x{H} h'={hp}: pooled events {len(ev)}; holes mean {ev[:,0].mean():.1f} max {ev[:,0].max()}; "
          f"levels top mean {ev[:,1].mean():.1f} max {ev[:,1].max()}; bottom mean {ev[:,2].mean():.1f} max {ev[:,2].max()}; "
          f"a mean {ev[:,5].mean():.1f}, b mean {ev[:,6].mean():.1f}")

# plan-loop sections (cycles): select (scan + warp min), record, unlink, refresh
for (W, H, hp, k, seed) in [(256, 256, 153, 39322, 257), (512, 512, 307, 157286, 0x51200000)]:
    occ = sample_grids(seed, 1, W, H, k)
    out = np.zeros(16, np.int64)
    lib.recon_debug_grid_phases(0, occ.ctypes.data_as(C.c_void_p), W, H, hp, out.ctypes.data_as(C.c_void_p), 16)
    print(f"plan {W}x{H}: select {out[8]/1965:.1f} us, record {out[9]/1965:.1f} us, unlink {out[10]/1965:.1f} us, "
          f"refresh {out[11]/1965:.1f} us")
