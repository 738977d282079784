"""Batching fixtures at C3 / C4 / C5 scale from the UNMODIFIED reference
(oracle/_ref/librecon_ref.so, built by oracle/Makefile from /root/reference).

Per instance: status, path_count, total_displacement, batch_count and the
digest64 of tests/digest.py (paths + the full move_batch).  The GPU suite
(tests/test_batching_scale_gpu.py) compares the B200 pipeline with these on
the GPU box, where /root/reference does not exist.

  python tests/golden/make_batch_scale.py [c3] [c4] [c5 N] [c5c N]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from digest import pipeline_digests  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

ref = ReconLib(os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so"), "ref")

# name: solver, W, H, h', atoms, seed0, preset, move stride
CASES = {
    "c3_none": ("bird", 64, 64, 40, 2662, 0x64000000, 0, 64 * 64 * 12),
    "c3_coldir": ("bird", 64, 64, 40, 2662, 0x64000000, 1, 64 * 64 * 12),
    "c4_none": ("redrec", 256, 256, 153, 39322, 0x25600000, 0, 1_500_000),
    "c4_coldir": ("redrec", 256, 256, 153, 39322, 0x25600000, 1, 1_500_000),
    "c5_none": ("bird", 512, 512, 307, 157286, 0x51200000, 0, 12_000_000),
    "c5_coldir": ("bird", 512, 512, 307, 157286, 0x51200000, 1, 12_000_000),
}


def run(name: str, count: int, chunk: int):
    solver, W, H, hp, k, seed0, preset, ms = CASES[name]
    cols = {key: [] for key in ("status", "path_count", "total_displacement", "batch_count", "digest")}
    t0 = time.time()
    for c0 in range(0, count, chunk):
        n = min(chunk, count - c0)
        occ = sample_grids(seed0 + c0, n, W, H, k)
        out = ref.pipeline_batch(solver, occ, n, W, H, hp, preset, ms)
        cols["digest"].append(pipeline_digests(out, n, W * hp, ms))
        for key in ("status", "path_count", "total_displacement", "batch_count"):
            cols[key].append(out[key].copy())
        print(f"{name}: {c0 + n}/{count} {time.time() - t0:.0f}s", flush=True)
    res = {key: np.concatenate(v) for key, v in cols.items()}
    res["case"] = np.array([W, H, hp, k, seed0, preset, ms, count], np.int64)
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), **res)


if __name__ == "__main__":
    args = sys.argv[1:] or ["c3_none", "c3_coldir", "c4_none", "c4_coldir", "c5_none", "64"]
    i = 0
    while i < len(args):
        name = args[i]
        count = 4096 if name.startswith("c3") else 8
        if i + 1 < len(args) and args[i + 1].isdigit():
            count = int(args[i + 1])
            i += 1
        chunk = 512 if name.startswith("c3") else 8
        run(name, count, chunk)
        i += 1
