"""Two half-chunks of C5 on two contexts (streams), issued back to back, vs one
chunk on one context: does the latency-bound leap phase of one half hide
behind the other half's solve / DAG / window kernels?

  python tools/overlap_probe.py [B] [steps]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import LIB_PATH  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402
from paper_2504_06182_b200.pipeline import C5, PipelineRunner  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wait = int(os.environ.get("OVERLAP_WAIT", "0"))
wl = C5
occ = sample_grids(wl.seed_base, B, wl.W, wl.H, wl.atoms)
wpc = (wl.H + 63) // 64
half = B // 2


def timed(runners, parts):
    torch.cuda.synchronize()
    for r, (o, n) in zip(runners, parts):
        r.load(occ[o * wl.W * wpc:(o + n) * wl.W * wpc], n)
    for _ in range(2):
        for r, (o, n) in zip(runners, parts):
            r.run(n, stats=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        for r, (o, n) in zip(runners, parts):
            r.run(n, stats=False)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e3


lib1 = ReconLib(LIB_PATH, "one")
r1 = PipelineRunner(lib1, wl, B)
ms1 = timed([r1], [(0, B)])
del r1
lib1.close()
torch.cuda.empty_cache()
libs = [ReconLib(LIB_PATH, "a"), ReconLib(LIB_PATH, "b")]
rs = [PipelineRunner(libs[0], wl, half), PipelineRunner(libs[1], wl, B - half)]
ms2 = timed(rs, [(0, half), (half, B - half)])
print({"B": B, "one_chunk_ms": ms1, "one_grids_s": B / ms1 * 1e3, "two_halves_ms": ms2, "two_grids_s": B / ms2 * 1e3})
