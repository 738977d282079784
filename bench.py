#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 atom-reconfiguration core.

Metric (BASELINE.json): "red-rec/bird solve µs per 256×256 grid; grids/sec at
1/2/4/8 B200".  The grids/sec clause is quoted on C5: bird + batching
(preset none, the reference default) on 512×512 grids, h'=307 (ε-critical),
157,286 atoms (ε=0.6), seeds 0x51200000 + global instance index, 65,536
instances sharded across 1/2/4/8 B200.

One step = one HBM-resident chunk of B C5 instances per GPU through the fused
device pipeline (recon_pipeline_batch_run: bird solve -> occupancy DAG ->
batching), inputs already in HBM.  value = grids/s over all ranks (weak
scaling: rank r owns instances [r*B, (r+1)*B); instances are independent, so
no collective runs on the data path — torch.distributed carries only the
timing max and the digest gather).  The full 65,536-instance job is 65,536/B
such steps per GPU count.

Same line: the phase breakdown (solve / DAG / wide batching in windows / warp batching,
CUDA events on the context stream), rooflines, the per-instance stats record
(digest64) of the chunk, e2e through the host-buffer C-ABI call
(recon_pipeline_batch_run_host: H2D of the grids and D2H of paths + batch
schedule inside the timed region), the compiled reference (oracle/_ref)
timed on this host's cores on a bounded sample, and the other BASELINE
configs (C4 single-grid latency, the 256² red-rec batch, C3, C2) as extra keys.

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

METRIC = "red-rec/bird solve µs per 256×256 grid; grids/sec at 1/2/4/8 B200"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so")
W = H = 512
HP = 307
ATOMS = 157286
SEED_BASE = 0x51200000
WPC = (H + 63) // 64  # u64 words per column
MOVE_STRIDE = 12_000_000  # > the largest C5 total displacement (10.82 M over the first 512 seeds)
WORKLOAD = (f"C5: bird + batching (preset none) on {W}x{H} grids, h'={HP}, {ATOMS} atoms (eps=0.6), "
            f"seeds {hex(SEED_BASE)} + global instance index")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


# ---- the reference arm: the compiled reference only (no repo .so is mapped) --------

def ref_inputs(ref_lib, first: int, count: int) -> np.ndarray:
    """Instances [first, first + count) from the reference's own generator,
    Rng(seed).sample_without_replacement (rng.hpp:49-59, exported by oracle/_ref
    as recon_ref_sample), packed into column-major occupancy bits."""
    import ctypes as C
    from paper_2504_06182_b200.inputs import pack_grid
    ref_lib.recon_ref_sample.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_void_p]
    ref_lib.recon_ref_sample.restype = None
    out = []
    v = np.zeros(ATOMS, np.int32)
    for i in range(count):
        ref_lib.recon_ref_sample(SEED_BASE + first + i, W * H, ATOMS, v.ctypes.data)
        occ2d = np.zeros((W, H), bool)
        occ2d[v // H, v % H] = True
        out.append(pack_grid(occ2d))
    return np.concatenate(out)


def cpu_reference(ref, occ: np.ndarray, count: int):
    """The compiled reference's bird + batch_moves on `count` C5 instances with
    every host thread (std::thread pool, one instance per task)."""
    cores = os.cpu_count() or 1
    os.environ["RECON_REF_THREADS"] = str(cores)
    t0 = time.perf_counter()
    out = ref.pipeline_batch("bird", occ, count, W, H, HP, 0, MOVE_STRIDE)
    dt = time.perf_counter() - t0
    return count / dt, cores, out


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    from paper_2504_06182_b200.abi import ReconLib
    ref = ReconLib(REF_LIB, "ref")
    cores = os.cpu_count() or 1
    sample = args.ref_sample or cores
    occ = ref_inputs(ref.lib, 0, sample)
    vals = []
    for i in range(args.warmup + args.steps):
        v, cores, _ = cpu_reference(ref, occ, sample)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.median(vals)
    line = {
        "metric": METRIC, "value": v, "unit": "grids/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * sample / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "batch_per_step": sample,
                   "sample": f"the first {sample} instances of the GPU arm's chunk (bounded CPU sample)"},
        "cpu_baseline": {"value": v, "unit": "grids/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
                         "sample": f"{sample} C5 instances per step, bird + batch_moves of the compiled reference "
                                   f"(oracle/_ref), std::thread pool over {cores} host threads"},
        "e2e": {"value": v, "unit": "grids/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- extra configs (informative; the headline is C5) --------------------------------

def other_configs(lib, torch, dev, stream):
    import ctypes as C
    from paper_2504_06182_b200.abi import ChainBatch, GridBatch
    from paper_2504_06182_b200.inputs import sample_chains, sample_grids
    from paper_2504_06182_b200.pipeline import C3, C4, PipelineRunner

    def timed(fn, reps=3, warm=1):
        for _ in range(warm):
            fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = fn()
            e1.record(stream)
            e1.synchronize()
            if st not in (None, 0):
                raise RuntimeError(f"config run failed {st}: {lib.last_cuda_error()}")
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    out = {}
    # C4: red-rec on one 256x256 grid, one instance per launch (latency)
    Wg = Hg = 256
    lat = {}
    for hp, seed in ((128, 256), (153, 257)):
        o1 = torch.from_numpy(sample_grids(seed, 1, Wg, Hg, 39322).view(np.int64)).to(dev)
        S = Wg * hp
        bufs = [torch.empty(S, dtype=torch.int32, device=dev) for _ in range(2)]
        i64 = torch.empty(1, dtype=torch.int64, device=dev)
        i32 = torch.empty(3, dtype=torch.int32, device=dev)
        g1 = GridBatch(o1.data_ptr(), 1, Wg, Hg, hp, bufs[0].data_ptr(), bufs[1].data_ptr(), None, i32.data_ptr(),
                       i64.data_ptr(), i32.data_ptr() + 4, i32.data_ptr() + 8, None)
        for solver, fn in (("redrec", lib.lib.recon_redrec_solve_batch), ("bird", lib.lib.recon_bird_solve_batch)):
            lat[f"{solver}_h{hp}_seed{seed}_us"] = 1000.0 * timed(lambda: fn(lib.ctx(), C.byref(g1)), reps=5, warm=3)
    out["c4_single_grid_latency"] = lat
    # the 256x256 red-rec / bird batch (round 1's headline): 2,048 grids h'153
    B = 2048
    occ = torch.from_numpy(sample_grids(0x25600000, B, Wg, Hg, 39322).view(np.int64)).to(dev)
    S = Wg * 153
    src = torch.empty(B * S, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    i64 = torch.empty(B, dtype=torch.int64, device=dev)
    i32 = torch.empty(3 * B, dtype=torch.int32, device=dev)
    gb = GridBatch(occ.data_ptr(), B, Wg, Hg, 153, src.data_ptr(), dst.data_ptr(), None, i32.data_ptr(), i64.data_ptr(),
                   i32.data_ptr() + 4 * B, i32.data_ptr() + 8 * B, None)
    for solver, fn in (("redrec", lib.lib.recon_redrec_solve_batch), ("bird", lib.lib.recon_bird_solve_batch)):
        ms = timed(lambda: fn(lib.ctx(), C.byref(gb)))
        out[f"{solver}_256x256_h153_batch2048"] = {"ms": ms, "grids_per_s": B / ms * 1e3, "us_per_grid": ms * 1e3 / B}
    del occ, src, dst
    # C3: bird + batching on 4,096 64x64 grids; C4 red-rec + batching
    for wl, n in ((C3, 4096), (C4, 64)):
        r = PipelineRunner(lib, wl, n)
        r.load(sample_grids(wl.seed_base, n, wl.W, wl.H, wl.atoms), n)
        ms = timed(lambda: r.run(n, stats=False))
        out[wl.name.split()[0].lower() + "_pipeline"] = {"instances": n, "ms": ms, "grids_per_s": n / ms * 1e3}
        del r
    # C2: 1M chains of 1024
    n, k, tl, th, cnt = 1024, 563, 256, 767, 1 << 20
    occ = torch.from_numpy(sample_chains(0x1D000000, cnt, n, k).view(np.int64)).to(dev)
    nt = th - tl + 1
    src = torch.empty(cnt * nt, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    i64 = torch.empty(cnt, dtype=torch.int64, device=dev)
    i32 = torch.empty(3 * cnt, dtype=torch.int32, device=dev)
    cb = ChainBatch(occ.data_ptr(), cnt, n, tl, th, src.data_ptr(), dst.data_ptr(), i64.data_ptr(), i32.data_ptr(),
                    i32.data_ptr() + 4 * cnt, i32.data_ptr() + 8 * cnt)
    ms = timed(lambda: lib.lib.recon_solve_1d_batch(lib.ctx(), C.byref(cb)))
    out["c2_1m_chains"] = {"ms": ms, "chains_per_s": cnt / ms * 1e3}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0,
                    help="C5 instances per GPU per step (one HBM-resident chunk; default: what HBM holds, <= 1536)")
    ap.add_argument("--e2e-batch", type=int, default=0, help="instances per e2e host-API step (default: the chunk)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=0, help="CPU sample (default: one instance per host thread)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e and the other configs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import ctypes as C

    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws > 1:
        # RECON_BENCH_BACKEND=gloo: functional runs with more ranks than GPUs
        backend = os.environ.get("RECON_BENCH_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    from paper_2504_06182_b200 import load_native
    from paper_2504_06182_b200.abi import STATS_DTYPE, GridBatch, PipelineBatch
    from paper_2504_06182_b200.inputs import sample_grids
    from paper_2504_06182_b200.pipeline import C5, PipelineRunner, algorithmic_bytes

    lib = load_native()
    lib.ctx(local)
    dev = torch.device("cuda", local)
    B = args.batch
    if not B:
        # the largest chunk HBM holds (device buffers + the library workspace
        # ~100 MB per instance), capped: the batching latency is paid once per step
        from paper_2504_06182_b200.pipeline import bytes_per_instance
        free, _ = torch.cuda.mem_get_info(dev)
        B = int(max(64, min(1536, (free - (6 << 30)) // bytes_per_instance(C5))) // 64 * 64)
    first = rank * B
    runner = PipelineRunner(lib, C5, B, device=local)
    stream = runner.stream
    occ_h = sample_grids(SEED_BASE + first, B, W, H, ATOMS)
    runner.load(occ_h, B)

    def step():
        runner.run(B, stats=False)

    # warm-up (W untimed steps), then K timed steps bracketed by barrier + sync
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.launch_count()
    times = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = lib.launch_count() - launches0  # every kernel of the library in the timed region
    if ws > 1:
        dist.barrier()
    ms = statistics.mean(times)
    if ws > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ws * B / (ms * 1e-3)

    # phase breakdown in separate steps (events between the phases)
    lib.set_kernel_timing(True)
    phases = []
    for _ in range(2):
        step()
        ph = (C.c_float * 4)()
        lib.lib.recon_ctx_phase_times(lib.ctx(), ph, 4)
        phases.append(list(ph))
    lib.set_kernel_timing(False)
    ph = [statistics.mean(p[i] for p in phases) for i in range(4)]
    solve_ms, dag_ms, wide_ms, warp_ms = ph

    # the chunk's per-instance stats record (digest64), outside the timed region
    runner.run(B, stats=True)
    st = runner.stats(B)
    ok = st["status"] == 0
    alg = algorithmic_bytes(st, C5)
    alg_solve = algorithmic_bytes(st, C5, batching=False)
    alg_sched = alg - alg_solve
    hbm, sm_max_mhz, peak_kind = peaks()
    batch_ms = wide_ms + warp_ms
    nb_mean = float(st["batch_count"][ok].mean()) if ok.any() else 0.0
    clocks = clk.summary()
    mhz = clocks.get("sm_mhz") or sm_max_mhz
    traffic = traffic_note = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get("c5_batching", {})
        if tr.get("per_instance_dram_bytes"):
            # DRAM bytes of the two batching kernels per instance (ncu --set full
            # at 64 instances) times this chunk
            traffic = tr["per_instance_dram_bytes"] * B
            traffic_note = (f"ncu dram read+write of both batching kernels, {tr['per_instance_dram_bytes'] / 1e6:.0f} MB "
                            f"per instance ({tr['source']}), x {B} instances")
    digests = st["digest"]
    job = {"instances": [first, first + B], "digest_sum": int(np.sum(digests, dtype=np.uint64)),
           "statuses": {str(k): int(v) for k, v in zip(*np.unique(st["status"], return_counts=True))}}
    if ws > 1:
        parts = [None] * ws
        dist.all_gather_object(parts, (first, digests.tolist(), st["status"].tolist()))
        if rank == 0:
            parts.sort()
            alld = np.array([d for p in parts for d in p[1]], np.uint64)
            job = {"instances": [0, ws * B], "digest_sum": int(np.sum(alld, dtype=np.uint64)),
                   "statuses": {str(k): int(v) for k, v in
                                zip(*np.unique(np.array([s for p in parts for s in p[2]]), return_counts=True))}}

    # e2e: the host-buffer C-ABI call over pinned host memory, H2D + D2H inside
    # the timed region: recon_pipeline_batch_run_host_runs (paths + the batch
    # schedule as runs), then the same with the per-move schedule on fewer
    # instances (e2e_move_batch)
    e2e = e2e_mb = None
    others = None
    if not args.no_extras:
        from paper_2504_06182_b200.abi import ScheduleRuns
        del runner
        torch.cuda.empty_cache()
        S = W * HP
        RST = S + 65536

        def host_call(E, runs_format):
            h_occ = torch.from_numpy(occ_h[: E * W * WPC].view(np.int64)).pin_memory()
            h_src = torch.empty(E * S, dtype=torch.int32).pin_memory()
            h_dst = torch.empty(E * S, dtype=torch.int32).pin_memory()
            h_i32 = torch.empty(4 * E, dtype=torch.int32).pin_memory()
            h_td = torch.empty(E, dtype=torch.int64).pin_memory()
            g = GridBatch(h_occ.data_ptr(), E, W, H, HP, h_src.data_ptr(), h_dst.data_ptr(), None, h_i32.data_ptr(),
                          h_td.data_ptr(), h_i32.data_ptr() + 4 * E, h_i32.data_ptr() + 8 * E, None)
            if runs_format:
                h_rs = torch.empty(2 * E * RST, dtype=torch.int32).pin_memory()
                h_rc = torch.empty(E, dtype=torch.int64).pin_memory()
                pb = PipelineBatch(g, 1, 0, MOVE_STRIDE, None, h_i32.data_ptr() + 12 * E)
                rr = ScheduleRuns(RST, h_rs.data_ptr(), h_rs.data_ptr() + 4 * E * RST, h_rc.data_ptr())
                call = lambda: lib.lib.recon_pipeline_batch_run_host_runs(lib.ctx(), C.byref(pb), C.byref(rr))  # noqa: E731
            else:
                h_mb = torch.empty(E * MOVE_STRIDE, dtype=torch.int32).pin_memory()
                pb = PipelineBatch(g, 1, 0, MOVE_STRIDE, h_mb.data_ptr(), h_i32.data_ptr() + 12 * E)
                call = lambda: lib.lib.recon_pipeline_batch_run_host(lib.ctx(), C.byref(pb))  # noqa: E731
            ts = []
            ke = max(2, min(args.steps, 3)) if runs_format else 1
            for i in range(2 + ke):
                t0 = time.perf_counter()
                r = call()
                dt = time.perf_counter() - t0
                if r != 0:
                    raise RuntimeError(f"host pipeline failed {r}: {lib.last_cuda_error()}")
                if i >= 2:
                    ts.append(dt)
            # the host call returns the device path's results (first instances of the chunk)
            assert np.array_equal(h_i32[E:2 * E].numpy(), st["status"][:E])
            assert np.array_equal(h_i32[3 * E:4 * E].numpy()[ok[:E]], st["batch_count"][:E][ok[:E]])
            sched = int(8 * h_rc.numpy().sum()) if runs_format else int(4 * h_td.numpy().clip(0)[ok[:E]].sum())
            return statistics.median(ts), int(E * S * 8 + E * 28 + sched)

        E = min(args.e2e_batch or B, B)
        e2e_s, d2h = host_call(E, True)
        mb_s, mb_d2h = host_call(min(128, E), False)
        if ws > 1:
            t = torch.tensor([e2e_s], device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": ws * E / e2e_s, "unit": "grids/s", "h2d_bytes_per_step": E * W * WPC * 8,
               "d2h_bytes_per_step": d2h, "instances_per_step": E,
               "call": "recon_pipeline_batch_run_host_runs (pinned host buffers): paths + the batch schedule as "
                       "runs of consecutive batch indices (recon_schedule_runs, lossless; tests expand it back)",
               "achieved_d2h_gbs": d2h / e2e_s / 1e9}
        e2e_mb = {"value": ws * min(128, E) / mb_s, "unit": "grids/s", "instances_per_step": min(128, E),
                  "d2h_bytes_per_step": mb_d2h,
                  "call": "recon_pipeline_batch_run_host (pinned): one int32 batch index per move copied back"}
        if rank == 0 and ws == 1:
            torch.cuda.empty_cache()
            others = other_configs(lib, torch, dev, stream)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from paper_2504_06182_b200.abi import ReconLib
        ref = ReconLib(REF_LIB, "ref")
        cores = os.cpu_count() or 1
        sample = args.ref_sample or cores
        v, cores, out = cpu_reference(ref, occ_h[: sample * W * WPC], sample)
        # the reference's outputs on the sample equal the device's
        assert np.array_equal(out["status"], st["status"][:sample])
        assert np.array_equal(out["batch_count"][ok[:sample]], st["batch_count"][:sample][ok[:sample]])
        cpu = {"value": v, "unit": "grids/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
               "sample": f"first {sample} instances of the chunk, bird + batch_moves of the compiled reference "
                         f"(oracle/_ref), std::thread pool over {cores} host threads; statuses and batch counts "
                         f"equal the device's"}

    if rank == 0:
        step_s = ms * 1e-3
        line = {
            "metric": METRIC, "value": value, "unit": "grids/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch_per_gpu_per_step": B,
                       "step": "one HBM-resident chunk per GPU: recon_pipeline_batch_run (solve -> DAG -> batching)",
                       "job": f"65,536 instances = {65536 // (ws * B)} steps at {ws} GPU(s)",
                       "parallelism": f"instances sharded over {ws} GPU(s), no collective on the data path",
                       "l2": "no flush: a chunk's inputs + outputs + workspace (~100 GB) dwarf the 126 MB L2"},
            "us_per_grid": ms * 1000.0 / B,
            "gpu_launches": launches,
            "phases_ms": {"solve": solve_ms, "dag": dag_ms, "batching_wide": wide_ms, "batching_warp": warp_ms,
                          "note": "batching_wide: rb::batch_window_kernel (ready sets > 32); batching_warp: the leap "
                                  "kernel rb::batch_pipeline_kernel<16>"},
            "roofline": {
                "bound": "hbm", "achieved": alg_sched / (batch_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": alg_sched / (batch_ms * 1e-3) / 1e9 / hbm, "traffic": traffic, "traffic_source": traffic_note,
                "peak_kind": peak_kind,
                "kernel": "batching phase: rb::batch_window_kernel + rb::batch_pipeline_kernel<16> (leap)",
                "algorithmic_bytes_per_launch": alg_sched,
                "algorithmic_bytes_rule": "4 B per elementary move of the batch schedule (SURVEY §8(d) 4*D)",
                "kernel_ms": batch_ms,
                "whole_step": {"algorithmic_bytes": alg, "achieved_gbs": alg / step_s / 1e9,
                               "frac": alg / step_s / 1e9 / hbm,
                               "rule": "ceil(W*H/8) + 8*P + 32 + 4*D per instance (SURVEY §8(d)), P/D the instances' own"},
                "solve_phase": {"algorithmic_bytes": alg_solve, "ms": solve_ms,
                                "achieved_gbs": alg_solve / (solve_ms * 1e-3) / 1e9,
                                "frac": alg_solve / (solve_ms * 1e-3) / 1e9 / hbm},
                "latency": {"batches_per_instance": nb_mean,
                            "cycles_per_batch": batch_ms * 1e-3 * mhz * 1e6 / nb_mean if nb_mean else None,
                            "note": "batching phase time x SM clock / mean batch count: every instance of the chunk "
                                    "runs its dependent batch chain concurrently"}},
            "stats": job,
            "clocks": clocks,
        }
        if e2e:
            line["e2e"] = e2e
            line["e2e_move_batch"] = e2e_mb
        if cpu:
            line["cpu_baseline"] = cpu
        if others:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
