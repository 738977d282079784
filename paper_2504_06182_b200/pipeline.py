"""Chunked, device-resident driver of the fused pipeline: solve (red-rec or
bird) -> occupancy DAG -> batching (recon_pipeline_batch_run) -> per-instance
stats record with digest64 (recon_pipeline_stats).

A C5 job (65,536 instances of 512x512, ~10.7 M moves each) does not fit in
HBM at once: the output schedule alone is ~43 MB per instance.  The runner
owns one chunk's worth of device buffers and walks a job chunk by chunk
(SURVEY.md §7 (iv)); every rank of a sharded job runs its own contiguous
range (shard.py), so the per-instance stats are identical for any GPU count.
torch is only used for device memory and the stream; every kernel is the
native library's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .abi import STATS_DTYPE, GridBatch, PipelineBatch, words_per_column


@dataclass(frozen=True)
class Workload:
    name: str
    solver: str          # "redrec" | "bird"
    W: int
    H: int
    h_prime: int
    atoms: int
    seed_base: int
    preset: int          # 0 none, 1 column_direction
    move_stride: int     # >= the largest total displacement of an instance

    @property
    def paths(self) -> int:
        return self.W * self.h_prime


# BASELINE.json configs with batching
C3 = Workload("C3 bird+batching 64x64 h'40", "bird", 64, 64, 40, 2662, 0x64000000, 0, 64 * 64 * 12)
C4 = Workload("C4 red-rec+batching 256x256 h'153", "redrec", 256, 256, 153, 39322, 0x25600000, 0, 1_500_000)
C5 = Workload("C5 bird+batching 512x512 h'307", "bird", 512, 512, 307, 157286, 0x51200000, 0, 12_000_000)


def bytes_per_instance(wl: Workload) -> int:
    """Device memory of one instance: the runner's buffers plus the library's
    pipeline workspace (capi_batch.cu), rounded up."""
    S, WH = wl.paths, wl.W * wl.H
    outs = wl.W * words_per_column(wl.H) * 8 + 2 * S * 4 + wl.move_stride * 4 + 64
    # owner maps 32 B/vertex + coverage 8 B/vertex, i32 scratch 9*4 B/path,
    # i64 16 B/path, records 32 B/path, path records 16 B/path, bitmaps,
    # vmin 4 B/vertex, successor lists (~48 per path)
    work = 40 * WH + 36 * S + 16 * S + 32 * S + 16 * S + WH // 4 + 4 * WH + 48 * 4 * S
    return outs + work


class PipelineRunner:
    """Device buffers for `chunk` instances of one workload, on one GPU."""

    def __init__(self, lib, wl: Workload, chunk: int, device: int = 0, preset: int | None = None):
        import torch
        self.torch = torch
        self.lib = lib
        self.wl = wl
        self.chunk = chunk
        self.preset = wl.preset if preset is None else preset
        lib.ctx(device)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(lib.lib.recon_ctx_stream(lib.ctx()))
        S, wpc = wl.paths, words_per_column(wl.H)
        d = self.dev
        self.occ = torch.empty(chunk * wl.W * wpc, dtype=torch.int64, device=d)
        self.src = torch.empty(chunk * S, dtype=torch.int32, device=d)
        self.dst = torch.empty(chunk * S, dtype=torch.int32, device=d)
        self.pcount = torch.empty(chunk, dtype=torch.int32, device=d)
        self.tdisp = torch.empty(chunk, dtype=torch.int64, device=d)
        self.status = torch.empty(chunk, dtype=torch.int32, device=d)
        self.detail = torch.empty(chunk, dtype=torch.int32, device=d)
        self.mb = torch.empty(chunk * wl.move_stride, dtype=torch.int32, device=d)
        self.nb = torch.empty(chunk, dtype=torch.int32, device=d)
        self.stats_d = torch.empty(chunk * STATS_DTYPE.itemsize, dtype=torch.uint8, device=d)
        self.n = 0

    def _batch(self, n: int) -> PipelineBatch:
        wl = self.wl
        g = GridBatch(self.occ.data_ptr(), n, wl.W, wl.H, wl.h_prime, self.src.data_ptr(), self.dst.data_ptr(), None,
                      self.pcount.data_ptr(), self.tdisp.data_ptr(), self.status.data_ptr(),
                      self.detail.data_ptr(), None)
        return PipelineBatch(g, 1 if wl.solver == "bird" else 0, self.preset, wl.move_stride, self.mb.data_ptr(),
                             self.nb.data_ptr())

    def load(self, occ_host: np.ndarray, n: int) -> None:
        """Copies n instances' occupancy bits (host) into the chunk's input buffer."""
        t = self.torch.from_numpy(np.ascontiguousarray(occ_host).view(np.int64))
        with self.torch.cuda.stream(self.stream):
            self.occ[: t.numel()].copy_(t, non_blocking=False)
        self.n = n

    def run(self, n: int | None = None, stats: bool = True) -> None:
        """Enqueues the pipeline (and the stats record) for the loaded instances on the context stream."""
        n = self.n if n is None else n
        pb = self._batch(n)
        st = self.lib.lib.recon_pipeline_batch_run(self.lib.ctx(), C.byref(pb))
        self.lib._check(st, 0)
        if stats:
            st = self.lib.lib.recon_pipeline_stats(self.lib.ctx(), C.byref(pb), self.stats_d.data_ptr())
            self.lib._check(st, 0)

    def stats(self, n: int | None = None) -> np.ndarray:
        n = self.n if n is None else n
        self.stream.synchronize()
        raw = self.stats_d[: n * STATS_DTYPE.itemsize].cpu().numpy()
        return raw.view(STATS_DTYPE).copy()

    def outputs(self) -> dict:
        """Host copies of the chunk's outputs in the ReconLib.pipeline_batch layout."""
        self.stream.synchronize()
        n, S, ms = self.n, self.wl.paths, self.wl.move_stride
        return {"path_src": self.src[: n * S].cpu().numpy(), "path_dst": self.dst[: n * S].cpu().numpy(),
                "path_count": self.pcount[:n].cpu().numpy(), "total_displacement": self.tdisp[:n].cpu().numpy(),
                "status": self.status[:n].cpu().numpy(), "detail": self.detail[:n].cpu().numpy(),
                "batch_count": self.nb[:n].cpu().numpy(), "move_batch": self.mb[: n * ms].cpu().numpy()}

    def run_range(self, first: int, count: int) -> np.ndarray:
        """Stats of instances [first, first + count) of the workload (seeds
        seed_base + index), chunk by chunk."""
        from .inputs import sample_grids
        wl = self.wl
        out = np.zeros(count, STATS_DTYPE)
        for c0 in range(0, count, self.chunk):
            n = min(self.chunk, count - c0)
            self.load(sample_grids(wl.seed_base + first + c0, n, wl.W, wl.H, wl.atoms), n)
            self.run(n)
            out[c0:c0 + n] = self.stats(n)
        return out


def algorithmic_bytes(stats: np.ndarray, wl: Workload, batching: bool = True) -> int:
    """ceil(W*H/8) input bits + 8*P path list + 32 stats
    (+ 4*D batch schedule) per instance, from the instances' own outputs."""
    ok = stats["status"] == 0
    n = len(stats)
    b = n * ((wl.W * wl.H + 7) // 8) + 32 * n + 8 * int(stats["path_count"][ok].sum())
    if batching:
        b += 4 * int(stats["total_displacement"][ok].sum())
    return b
