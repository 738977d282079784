"""Runs one pipeline workload range on the GPU and prints its per-instance
status / batch count / digest64 as JSON (tests/test_batching_scale_gpu.py
runs it in a subprocess so that the kernel-variant overrides, which the
library reads once per process from the environment, can differ per run).

  RECON_BATCH_LEAP=0 python tests/scale_variant.py c5 0 160 [preset]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.pipeline import C3, C4, C5, PipelineRunner  # noqa: E402

WL = {"c3": C3, "c4": C4, "c5": C5}

if __name__ == "__main__":
    name, first, count = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    preset = int(sys.argv[4]) if len(sys.argv) > 4 else None
    lib = load_native()
    wl = WL[name]
    r = PipelineRunner(lib, wl, count, preset=preset)
    st = r.run_range(first, count)
    print(json.dumps({"status": st["status"].tolist(), "batch_count": st["batch_count"].tolist(),
                      "digest": [str(int(x)) for x in st["digest"]], "launches": lib.launch_count()}))
