"""Times each BASELINE config shape on the GPU (device-resident inputs, CUDA events).

  python tools/perf_probe.py [names...]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.abi import ChainBatch, GridBatch, PipelineBatch, ValidateBatch  # noqa: E402
from paper_2504_06182_b200.inputs import sample_chains, sample_grids  # noqa: E402

lib = load_native()
lib.ctx(0)
stream = torch.cuda.ExternalStream(lib.lib.recon_ctx_stream(lib.ctx()))
dev = torch.device("cuda", 0)


def timeit(fn, reps=3, warm=1):
    ts = []
    for i in range(warm + reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        if i >= warm:
            ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts)


def grid(solver, W, H, hp, k, seed, count):
    occ = torch.from_numpy(sample_grids(seed, count, W, H, k).view(np.int64)).to(dev)
    S = W * hp
    src = torch.empty(count * S, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    pc = torch.empty(count, dtype=torch.int32, device=dev)
    td = torch.empty(count, dtype=torch.int64, device=dev)
    st = torch.empty(count, dtype=torch.int32, device=dev)
    de = torch.empty(count, dtype=torch.int32, device=dev)
    b = GridBatch(occ.data_ptr(), count, W, H, hp, src.data_ptr(), dst.data_ptr(), None, pc.data_ptr(),
                  td.data_ptr(), st.data_ptr(), de.data_ptr(), None)
    fn = lib.lib.recon_redrec_solve_batch if solver == "redrec" else lib.lib.recon_bird_solve_batch
    mn, avg = timeit(lambda: fn(lib.ctx(), C.byref(b)))
    assert int((st != 0).sum()) == 0
    P = int(pc.sum())
    lib.set_kernel_timing(True)
    fn(lib.ctx(), C.byref(b))
    torch.cuda.synchronize()
    kt = lib.kernel_times()
    lib.set_kernel_timing(False)
    return {"ms": mn, "plan_ms": kt[0], "exec_ms": kt[1], "grids_per_s": count / mn * 1e3, "us_per_grid": mn * 1e3 / count,
            "paths_per_grid": P / count, "GBps_alg": (count * W * H / 8 + 8 * P + 32 * count) / mn / 1e6}


def pipeline(solver, W, H, hp, k, seed, count, preset, ms_=None, validate=False):
    occ = torch.from_numpy(sample_grids(seed, count, W, H, k).view(np.int64)).to(dev)
    S = W * hp
    src = torch.empty(count * S, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    pc = torch.empty(count, dtype=torch.int32, device=dev)
    td = torch.empty(count, dtype=torch.int64, device=dev)
    st = torch.empty(count, dtype=torch.int32, device=dev)
    de = torch.empty(count, dtype=torch.int32, device=dev)
    ms_ = ms_ or W * H * 12
    mb = torch.empty(count * ms_, dtype=torch.int32, device=dev)
    bc = torch.empty(count, dtype=torch.int32, device=dev)
    g = GridBatch(occ.data_ptr(), count, W, H, hp, src.data_ptr(), dst.data_ptr(), None, pc.data_ptr(),
                  td.data_ptr(), st.data_ptr(), de.data_ptr(), None)
    pb = PipelineBatch(g, 1 if solver == "bird" else 0, preset, ms_, mb.data_ptr(), bc.data_ptr())
    t0 = time.perf_counter()
    mn, avg = timeit(lambda: lib.lib.recon_pipeline_batch_run(lib.ctx(), C.byref(pb)), reps=2)
    D = int(td.sum())
    res = {"ms": mn, "grids_per_s": count / mn * 1e3, "moves_per_grid": D / count,
           "batches_per_grid": float(bc.float().mean()), "status_nonzero": int((st != 0).sum())}
    if validate:  # on-device validators over the whole batch (failed solves report path_count 0)
        verdict = torch.empty(count, dtype=torch.int32, device=dev)
        vb = ValidateBatch(occ.data_ptr(), count, W, H, hp, src.data_ptr(), dst.data_ptr(), S, pc.data_ptr(),
                           td.data_ptr(), pc.data_ptr(), 2, None, None, None, mb.data_ptr(), ms_, bc.data_ptr(),
                           preset, verdict.data_ptr())
        vmn, _ = timeit(lambda: lib.lib.recon_validate_batch_run(lib.ctx(), C.byref(vb)), reps=1)
        ok = st == 0
        res["validate_ms"] = vmn
        res["validate_pass"] = int(((verdict == 0) & ok).sum())
        res["validate_checked"] = int(ok.sum())
    return res


def chains(n, k, tl, th, seed, count):
    occ = torch.from_numpy(sample_chains(seed, count, n, k).view(np.int64)).to(dev)
    nt = th - tl + 1
    src = torch.empty(count * nt, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    td = torch.empty(count, dtype=torch.int64, device=dev)
    ds = torch.empty(count, dtype=torch.int32, device=dev)
    st = torch.empty(count, dtype=torch.int32, device=dev)
    de = torch.empty(count, dtype=torch.int32, device=dev)
    b = ChainBatch(occ.data_ptr(), count, n, tl, th, src.data_ptr(), dst.data_ptr(), td.data_ptr(), ds.data_ptr(),
                   st.data_ptr(), de.data_ptr())
    mn, avg = timeit(lambda: lib.lib.recon_solve_1d_batch(lib.ctx(), C.byref(b)))
    assert int((st != 0).sum()) == 0, "chain batch failed"
    bytes_ = count * (n // 8 + 8 * nt + 32)
    return {"ms": mn, "chains_per_s": count / mn * 1e3, "GBps_alg": bytes_ / mn / 1e6,
            "frac_hbm": bytes_ / mn / 1e6 / 6465.8}


def json_case(solver, W, H, hp, k, seed, preset, ms_):
    """solution + batch-schedule JSON of one pipeline instance, formatted on the device."""
    occ = torch.from_numpy(sample_grids(seed, 1, W, H, k).view(np.int64)).to(dev)
    S = W * hp
    src = torch.empty(S, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    pc = torch.empty(1, dtype=torch.int32, device=dev)
    td = torch.empty(1, dtype=torch.int64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    de = torch.empty(1, dtype=torch.int32, device=dev)
    mb = torch.empty(ms_, dtype=torch.int32, device=dev)
    bc = torch.empty(1, dtype=torch.int32, device=dev)
    g = GridBatch(occ.data_ptr(), 1, W, H, hp, src.data_ptr(), dst.data_ptr(), None, pc.data_ptr(),
                  td.data_ptr(), st.data_ptr(), de.data_ptr(), None)
    pb = PipelineBatch(g, 1 if solver == "bird" else 0, preset, ms_, mb.data_ptr(), bc.data_ptr())
    assert lib.lib.recon_pipeline_batch_run(lib.ctx(), C.byref(pb)) == 0
    torch.cuda.synchronize()
    P, D, nb = int(pc.item()), int(td.item()), int(bc.item())
    n = C.c_int64(0)
    lib.lib.recon_solution_json(lib.ctx(), W, H, P, src.data_ptr(), dst.data_ptr(), None, 0, None, None, P, D,
                                None, 0, C.byref(n))
    out = torch.empty(n.value, dtype=torch.uint8, device=dev)
    f = lambda: lib.lib.recon_solution_json(lib.ctx(), W, H, P, src.data_ptr(), dst.data_ptr(), None, 0, None, None,
                                            P, D, out.data_ptr(), n.value, C.byref(n))
    ms1, _ = timeit(f)
    nb_ = C.c_int64(0)
    lib.lib.recon_batch_schedule_json(lib.ctx(), W, H, P, src.data_ptr(), dst.data_ptr(), mb.data_ptr(), nb, preset,
                                      None, 0, C.byref(nb_))
    out2 = torch.empty(nb_.value, dtype=torch.uint8, device=dev)
    f2 = lambda: lib.lib.recon_batch_schedule_json(lib.ctx(), W, H, P, src.data_ptr(), dst.data_ptr(), mb.data_ptr(),
                                                   nb, preset, out2.data_ptr(), nb_.value, C.byref(nb_))
    ms2, _ = timeit(f2)
    return {"solution_json_MB": n.value / 1e6, "solution_json_ms": ms1, "solution_json_GBps": n.value / ms1 / 1e6,
            "batch_json_MB": nb_.value / 1e6, "batch_json_ms": ms2, "batch_json_GBps": nb_.value / ms2 / 1e6}


CASES = {
    "c4_json": lambda: json_case("redrec", 256, 256, 153, 39322, 257, 0, 1_500_000),
    "c5_json": lambda: json_case("bird", 512, 512, 307, 157286, 0x51200000, 0, 12_000_000),
    "c1_redrec": lambda: grid("redrec", 32, 32, 16, 614, 1, 4096),
    "c1_bird": lambda: grid("bird", 32, 32, 16, 614, 1, 4096),
    "c1_redrec_1": lambda: grid("redrec", 32, 32, 16, 614, 1, 1),
    "c4_redrec_h128_1": lambda: grid("redrec", 256, 256, 128, 39322, 256, 1),
    "c4_redrec_h153_1": lambda: grid("redrec", 256, 256, 153, 39322, 257, 1),
    "c4_bird_h153_1": lambda: grid("bird", 256, 256, 153, 39322, 257, 1),
    "c4_redrec_2048": lambda: grid("redrec", 256, 256, 153, 39322, 0x25600000, 2048),
    "c4_bird_2048": lambda: grid("bird", 256, 256, 153, 39322, 0x25600000, 2048),
    "r256_redrec_b2048": lambda: grid("redrec", 256, 256, 153, 39322, 0x25600000, 2048),
    "r256_bird_b2048": lambda: grid("bird", 256, 256, 153, 39322, 0x25600000, 2048),
    "r256_redrec_b1776": lambda: grid("redrec", 256, 256, 153, 39322, 0x25600000, 1776),
    "r256_redrec_b2368": lambda: grid("redrec", 256, 256, 153, 39322, 0x25600000, 2368),
    "r256_redrec_b8192": lambda: grid("redrec", 256, 256, 153, 39322, 0x25600000, 8192),
    "r256_bird_b8192": lambda: grid("bird", 256, 256, 153, 39322, 0x25600000, 8192),
    "r128_bird_b4096": lambda: grid("bird", 128, 128, 77, 9830, 0x12800000, 4096),
    "r128_redrec_b4096": lambda: grid("redrec", 128, 128, 77, 9830, 0x12800000, 4096),
    "c3_bird_solve": lambda: grid("bird", 64, 64, 40, 2662, 0x64000000, 4096),
    "c3_redrec_solve": lambda: grid("redrec", 64, 64, 40, 2662, 0x64000000, 4096),
    "r128_redrec_b4096": lambda: grid("redrec", 128, 128, 76, 9830, 0x12800000, 4096),
    "r128_bird_b4096": lambda: grid("bird", 128, 128, 76, 9830, 0x12800000, 4096),
    "c3_pipeline_none": lambda: pipeline("bird", 64, 64, 40, 2662, 0x64000000, 4096, 0),
    "c3_pipeline_coldir": lambda: pipeline("bird", 64, 64, 40, 2662, 0x64000000, 1024, 1),
    "c5_pipeline_512": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 512, 0, 11_000_000),
    "c5_pipeline_256": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 256, 0, 11_000_000),
    "c5_pipeline_4": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 4, 0, 12_000_000),
    "c5_pipeline_64": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 64, 0, 12_000_000),
    "c5_pipeline_1024": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 1024, 0, 12_000_000),
    "c5_pipeline_64_validate": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 64, 0, 12_000_000, True),
    "c5_pipeline_4_validate": lambda: pipeline("bird", 512, 512, 307, 157286, 0x51200000, 4, 0, 12_000_000, True),
    "c3_pipeline_validate": lambda: pipeline("bird", 64, 64, 40, 2662, 0x64000000, 4096, 0, None, True),
    "c4_pipeline_redrec_64_validate": lambda: pipeline("redrec", 256, 256, 153, 39322, 257, 64, 0, 1_500_000, True),
    "c4_pipeline_redrec_64": lambda: pipeline("redrec", 256, 256, 153, 39322, 257, 64, 0, 1_500_000),
    "c5_bird_solve_64": lambda: grid("bird", 512, 512, 307, 157286, 0x51200000, 64),
    "c5_bird_solve_512": lambda: grid("bird", 512, 512, 307, 157286, 0x51200000, 512),
    "c5_bird_solve_1": lambda: grid("bird", 512, 512, 307, 157286, 0x51200000, 1),
    "c2_chains_1m": lambda: chains(1024, 563, 256, 767, 0x1D000000, 1 << 20),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nme in names:
        t0 = time.time()
        try:
            r = CASES[nme]()
        except Exception as e:  # noqa: BLE001
            r = {"error": repr(e)}
        r["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps({nme: r}), flush=True)
