"""Run-length schedule format (recon_schedule_runs): lossless against the
per-move batch indices, on the CPU checkers (here) and on the device
(tests/test_batching_scale_gpu.py, tests/test_batching_gpu.py)."""
import numpy as np

from paper_2504_06182_b200.abi import expand_runs
from paper_2504_06182_b200.inputs import sample_grids


def test_oracle_runs_expand_to_move_batch(oracle):
    W = H = 32
    occ = sample_grids(1, 6, W, H, 614)
    ms = W * H * 12
    for solver in ("redrec", "bird"):
        for preset in (0, 1):
            o = oracle.pipeline_batch(solver, occ, 6, W, H, 16, preset, ms)
            r = oracle.pipeline_batch_runs(solver, occ, 6, W, H, 16, preset, ms)
            assert np.array_equal(r["status"], o["status"])
            rs = r["run_stride"]
            for i in range(6):
                D = int(o["total_displacement"][i])
                n = int(r["run_count"][i])
                got = expand_runs(r["run_slot"][i * rs:], r["run_batch"][i * rs:], n, D)
                assert np.array_equal(got, o["move_batch"][i * ms:i * ms + D])
                # maximal runs: consecutive runs never continue each other
                s, b = r["run_slot"][i * rs:i * rs + n], r["run_batch"][i * rs:i * rs + n]
                assert s[0] == 0 and (np.diff(s) > 0).all()
                assert not np.any(b[1:] == b[:-1] + np.diff(s))
