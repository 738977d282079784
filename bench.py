#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 atom-reconfiguration core.

Metric (BASELINE.json): "red-rec/bird solve µs per 256×256 grid; grids/sec at
1/2/4/8 B200".  One step = one batched red-rec solve (recon_redrec_solve_batch)
of B independent 256×256 grids, h'=153 (ε-critical: ~113 deficit columns, the
pairing loop runs), 39,322 atoms each (ε=0.6), seeds 0x25600000 + global index,
all resident in HBM.  value = grids/s over all ranks (weak scaling: each rank
solves its own B grids; instances are independent, so no collective runs on
the data path — torch.distributed only carries the timing max).

Side measurements on the same line: bird on the same grids, single-grid
latency (µs) for red-rec at h'=128 / 153 (C4), the roofline of the solve
kernel against MEASURED_PEAKS.json, e2e through the host-buffer C-ABI call
(recon_redrec_solve_batch_host: H2D of the grids + D2H of the paths inside the
timed region), and the reference CPU implementation (oracle/_ref, compiled
from the reference's own sources) timed on this host.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W = H = 256
HP = 153
ATOMS = 39322
SEED_BASE = 0x25600000
METRIC = "red-rec/bird solve µs per 256×256 grid; grids/sec at 1/2/4/8 B200"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def gen_inputs(rank: int, batch: int):
    from paper_2504_06182_b200.inputs import sample_grids
    return sample_grids(SEED_BASE + rank * batch, batch, W, H, ATOMS)


def algorithmic_bytes(path_counts: np.ndarray) -> int:
    # B = ceil(W*H/8) input bits + 8*P path list + 32 stats (no batching here)
    n = len(path_counts)
    return int(n * (W * H // 8) + 8 * int(path_counts.sum()) + 32 * n)


def cpu_reference(occ: np.ndarray, count: int, solver: str = "redrec"):
    """Times the compiled reference (oracle/_ref) on `count` grids with every host thread."""
    from paper_2504_06182_b200.abi import ReconLib
    ref = ReconLib(REF_LIB, "ref")
    cores = os.cpu_count() or 1
    os.environ["RECON_REF_THREADS"] = str(cores)
    wpc = (H + 63) // 64
    sub = np.ascontiguousarray(occ[: count * W * wpc])
    t0 = time.perf_counter()
    out = ref.grid_solve_batch(solver, sub, count, W, H, HP, host=True, with_events=False)
    dt = time.perf_counter() - t0
    assert (out["status"] == 0).all()
    return count / dt, cores, out


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    sample = args.ref_sample
    occ = gen_inputs(0, sample)
    vals = []
    for i in range(args.warmup + args.steps):
        v, cores, _ = cpu_reference(occ, sample)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.median(vals)
    line = {
        "metric": METRIC, "value": v, "unit": "grids/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * sample / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"red-rec {W}x{H} h'={HP} {ATOMS} atoms, batch of {sample} per step (bounded CPU sample)",
                   "seeds": hex(SEED_BASE)},
        "cpu_baseline": {"value": v, "unit": "grids/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample} grids per step, std::thread pool over all host threads"},
        "e2e": {"value": v, "unit": "grids/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def other_configs(lib, torch, dev, stream, reps=3):
    """C2 (1M chains of 1024, band [256, 767]) and C3 (4096 bird 64x64 h'40 +
    batching, preset none), each timed over `reps` runs after one warm-up."""
    import ctypes as C
    from paper_2504_06182_b200.abi import ChainBatch, GridBatch, PipelineBatch
    from paper_2504_06182_b200.inputs import sample_chains, sample_grids

    def run(fn):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = fn()
            e1.record(stream)
            e1.synchronize()
            if st != 0:
                raise RuntimeError(f"config run failed {st}: {lib.last_cuda_error()}")
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    out = {}
    n, k, tl, th, cnt = 1024, 563, 256, 767, 1 << 20
    occ = torch.from_numpy(sample_chains(0x1D000000, cnt, n, k).view(np.int64)).to(dev)
    nt = th - tl + 1
    src = torch.empty(cnt * nt, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    i64 = torch.empty(cnt, dtype=torch.int64, device=dev)
    i32 = torch.empty(3 * cnt, dtype=torch.int32, device=dev)
    cb = ChainBatch(occ.data_ptr(), cnt, n, tl, th, src.data_ptr(), dst.data_ptr(), i64.data_ptr(), i32.data_ptr(),
                    i32.data_ptr() + 4 * cnt, i32.data_ptr() + 8 * cnt)
    ms = run(lambda: lib.lib.recon_solve_1d_batch(lib.ctx(), C.byref(cb)))
    out["c2_1m_chains"] = {"ms": ms, "chains_per_s": cnt / ms * 1e3}
    del occ, src, dst, i64, i32
    W = H = 64
    cnt = 4096
    occ = torch.from_numpy(sample_grids(0x64000000, cnt, W, H, 2662).view(np.int64)).to(dev)
    S, mst = W * 40, W * H * 12
    src = torch.empty(cnt * S, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    td = torch.empty(cnt, dtype=torch.int64, device=dev)
    i32 = torch.empty(4 * cnt, dtype=torch.int32, device=dev)
    mb = torch.empty(cnt * mst, dtype=torch.int32, device=dev)
    g = GridBatch(occ.data_ptr(), cnt, W, H, 40, src.data_ptr(), dst.data_ptr(), None, i32.data_ptr(), td.data_ptr(),
                  i32.data_ptr() + 4 * cnt, i32.data_ptr() + 8 * cnt, None)
    pb = PipelineBatch(g, 1, 0, mst, mb.data_ptr(), i32.data_ptr() + 12 * cnt)
    ms = run(lambda: lib.lib.recon_pipeline_batch_run(lib.ctx(), C.byref(pb)))
    out["c3_bird_batching_4096"] = {"ms": ms, "grids_per_s": cnt / ms * 1e3}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=2048, help="grids per GPU per step")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2 / C3 side measurements")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws > 1:
        # RECON_BENCH_BACKEND=gloo: functional runs with more ranks than GPUs
        # (NCCL refuses two ranks on one device); timing values then mean nothing
        backend = os.environ.get("RECON_BENCH_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    from paper_2504_06182_b200 import load_native
    from paper_2504_06182_b200.abi import GridBatch
    import ctypes as C

    lib = load_native()
    lib.ctx(local)
    stream_ptr = lib.lib.recon_ctx_stream(lib.ctx())
    stream = torch.cuda.ExternalStream(stream_ptr)

    B = args.batch
    wpc = (H + 63) // 64
    occ_h = gen_inputs(rank, B)
    dev = torch.device("cuda", local)
    occ_d = torch.from_numpy(occ_h.view(np.int64)).to(dev)
    stride = W * HP
    bufs = {k: torch.empty(B * stride, dtype=torch.int32, device=dev) for k in ("src", "dst")}
    pcount = torch.empty(B, dtype=torch.int32, device=dev)
    tdisp = torch.empty(B, dtype=torch.int64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    detail = torch.empty(B, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def batch_struct():
        return GridBatch(occ_d.data_ptr(), B, W, H, HP, bufs["src"].data_ptr(), bufs["dst"].data_ptr(), None,
                         pcount.data_ptr(), tdisp.data_ptr(), status.data_ptr(), detail.data_ptr(), None)

    gb = batch_struct()

    def solve(fn):
        st = fn(lib.ctx(), C.byref(gb))
        if st != 0:
            raise RuntimeError(f"solve failed {st}: {lib.last_cuda_error()}")

    ktimes = []  # (planner ms, executor ms) per timed step, CUDA events on the context stream

    def timed(fn, steps, warmup, kernels=False):
        times = []
        lib.set_kernel_timing(kernels)
        for i in range(warmup + steps):
            with torch.cuda.stream(stream):
                flush.fill_(i)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            solve(fn)
            e1.record(stream)
            e1.synchronize()
            if i >= warmup:
                times.append(e0.elapsed_time(e1))
                if kernels:
                    ktimes.append(lib.kernel_times())
        lib.set_kernel_timing(False)
        return times

    # warm-up + correctness status
    solve(lib.lib.recon_redrec_solve_batch)
    torch.cuda.synchronize()
    assert int((status != 0).sum()) == 0, "solver statuses"

    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.launch_count()
    with Clocks(local) as clk:
        times = timed(lib.lib.recon_redrec_solve_batch, args.steps, args.warmup)
    launches = lib.launch_count() - launches0
    # per-kernel breakdown in a separate pass: events between the planner and
    # the executor serialise them (no programmatic dependent launch), so the
    # headline above is timed without them
    timed(lib.lib.recon_redrec_solve_batch, args.steps, args.warmup, kernels=True)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms = sum(times) / len(times)
    if ws > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    counts = pcount.cpu().numpy()
    alg_bytes = algorithmic_bytes(counts)
    hbm_peak, peak_kind = peaks()
    plan_ms = sum(k[0] for k in ktimes) / len(ktimes)
    exec_ms = sum(k[1] for k in ktimes) / len(ktimes)
    achieved_gbs = alg_bytes / (exec_ms * 1e-3) / 1e9  # dominant kernel: the executor
    traffic = warp_inst = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get("redrec_kernel", {})
        if tr.get("batch") == B and tr.get("workload_seed") == hex(SEED_BASE):
            traffic = tr.get("dram_bytes")
            warp_inst = tr.get("warp_inst")
    value = ws * B / (ms * 1e-3)

    # bird on the same grids (secondary)
    bird_times = timed(lib.lib.recon_bird_solve_batch, max(2, args.steps // 2), 1)
    bird_ms = sum(bird_times) / len(bird_times)

    # e2e through the host-buffer C-ABI call (pinned host memory)
    pin = {k: torch.empty(B * stride, dtype=torch.int32).pin_memory() for k in ("src", "dst")}
    occ_pin = torch.from_numpy(occ_h.view(np.int64)).pin_memory()
    h_cnt = torch.empty(B, dtype=torch.int32).pin_memory()
    h_td = torch.empty(B, dtype=torch.int64).pin_memory()
    h_st = torch.empty(B, dtype=torch.int32).pin_memory()
    h_det = torch.empty(B, dtype=torch.int32).pin_memory()
    hb = GridBatch(occ_pin.data_ptr(), B, W, H, HP, pin["src"].data_ptr(), pin["dst"].data_ptr(), None,
                   h_cnt.data_ptr(), h_td.data_ptr(), h_st.data_ptr(), h_det.data_ptr(), None)
    e2e = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        st = lib.lib.recon_redrec_solve_batch_host(lib.ctx(), C.byref(hb))
        dt = time.perf_counter() - t0
        assert st == 0
        if i >= args.warmup:
            e2e.append(dt)
    e2e_s = statistics.median(e2e)
    # the same call with the packed path list (src | dst << 16, 4 bytes per
    # path over the host link instead of 8): the headline e2e
    packed_pin = torch.empty(B * stride, dtype=torch.int32).pin_memory()
    cnt_unpacked = h_cnt.clone()
    hp_b = GridBatch(occ_pin.data_ptr(), B, W, H, HP, None, None, None,
                     h_cnt.data_ptr(), h_td.data_ptr(), h_st.data_ptr(), h_det.data_ptr(), None)
    e2e_p = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        st = lib.lib.recon_redrec_solve_batch_host_packed(lib.ctx(), C.byref(hp_b), packed_pin.data_ptr())
        dt = time.perf_counter() - t0
        assert st == 0
        if i >= args.warmup:
            e2e_p.append(dt)
    # same paths as the unpacked call (first and last instance)
    assert torch.equal(cnt_unpacked, h_cnt)
    for i in (0, B - 1):
        c0, n0 = i * stride, int(h_cnt[i])
        pk = packed_pin[c0:c0 + n0]
        assert torch.equal(pk & 0xFFFF, pin["src"][c0:c0 + n0]) and torch.equal((pk >> 16) & 0xFFFF, pin["dst"][c0:c0 + n0])
    e2e_p_s = statistics.median(e2e_p)
    # the host link's own device-to-host rate into pinned memory (the bound of
    # the e2e call): one copy of the packed path lists' size, CUDA events
    link = []
    dsrc = bufs["src"].view(torch.int32)
    for i in range(4):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            packed_pin.copy_(dsrc, non_blocking=True)
            e1.record(stream)
        e1.synchronize()
        if i:
            link.append(packed_pin.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    link_gbs = statistics.median(link)
    if ws > 1:
        t = torch.tensor([e2e_s, e2e_p_s], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, e2e_p_s = float(t[0].item()), float(t[1].item())
    h2d = B * W * wpc * 8
    d2h = B * stride * 4 * 2 + B * (4 + 8 + 4 + 4)
    d2h_p = B * stride * 4 + B * (4 + 8 + 4 + 4)

    # single-grid latency (C4: one instance per launch)
    lat = {}
    for hp, seed in ((128, 256), (153, 257)):
        from paper_2504_06182_b200.inputs import sample_grids
        o1 = torch.from_numpy(sample_grids(seed, 1, W, H, ATOMS).view(np.int64)).to(dev)
        g1 = GridBatch(o1.data_ptr(), 1, W, H, hp, bufs["src"].data_ptr(), bufs["dst"].data_ptr(), None,
                       pcount.data_ptr(), tdisp.data_ptr(), status.data_ptr(), detail.data_ptr(), None)
        ts = []
        for i in range(8):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            assert lib.lib.recon_redrec_solve_batch(lib.ctx(), C.byref(g1)) == 0
            e1.record(stream)
            e1.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1000.0)
        lat[f"h{hp}_seed{seed}_us"] = statistics.median(ts)

    # the other BASELINE configs at their own sizes (device-resident inputs,
    # CUDA events on the context stream; informative, the headline is above)
    others = None
    if rank == 0 and ws == 1 and not args.no_configs:
        others = other_configs(lib, torch, dev, stream)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        v, cores, _ = cpu_reference(occ_h, args.ref_sample)
        cpu = {"value": v, "unit": "grids/s", "cores": cores, "kind": "reference",
               "sample": f"first {args.ref_sample} grids of the batch, compiled reference red_rec "
                         f"(oracle/_ref), std::thread pool over all host threads"}

    # the executor is latency / issue bound, not HBM bound: its instruction
    # issue rate against the SMs' peak (4 warp-instructions per SM per clock)
    # says how close it runs to that ceiling
    issue = None
    clocks = clk.summary()
    if warp_inst and clocks.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_i = sms * 4 * clocks["sm_mhz"] * 1e6
        ach_i = warp_inst / (exec_ms * 1e-3)
        issue = {"warp_inst_per_launch": warp_inst, "achieved_ginst_s": ach_i / 1e9, "peak_ginst_s": peak_i / 1e9,
                 "frac": ach_i / peak_i, "source": "ncu smsp__inst_executed.sum of the same launch (profiles/traffic.json)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "grids/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"red-rec {W}x{H} h'={HP}, {ATOMS} atoms (eps=0.6), batch {B} grids/GPU/step",
                       "seeds": f"{hex(SEED_BASE)} + global index", "parallelism": f"instances sharded over {ws} GPU(s)",
                       "l2": "flushed between steps (256 MiB write)"},
            "us_per_grid": ms * 1000.0 / B,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "rb::redrec_kernel (executor)", "kernel_ms": exec_ms,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "planner_kernel_ms": plan_ms, "issue": issue},
            "e2e": {"value": ws * B / e2e_p_s, "unit": "grids/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h_p, "call": "recon_redrec_solve_batch_host_packed (pinned host buffers)",
                    "path_format": "u32 src | dst << 16 per path",
                    "link_d2h_gbs": link_gbs, "achieved_d2h_gbs": d2h_p / e2e_p_s / 1e9,
                    "link_frac": d2h_p / e2e_p_s / 1e9 / link_gbs},
            "e2e_unpacked": {"value": ws * B / e2e_s, "unit": "grids/s", "h2d_bytes_per_step": h2d,
                             "d2h_bytes_per_step": d2h, "call": "recon_redrec_solve_batch_host (pinned host buffers)",
                             "path_format": "i32 path_src[] + i32 path_dst[]"},
            "bird": {"grids_per_s": ws * B / (bird_ms * 1e-3), "ms_per_step": bird_ms},
            "latency_single_grid": lat,
            "other_configs": others,
            "clocks": clocks,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
