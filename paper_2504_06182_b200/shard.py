"""Multi-GPU sharding of independent instances.

Instances are independent pure functions of their seed, so a job is split
into contiguous per-rank ranges [g*N/G, (g+1)*N/G) and every rank runs its
range on its own GPU, chunk by chunk (pipeline.PipelineRunner); there is no
collective on the data path.  torch.distributed only carries the final host
gather of the per-instance stats records (status, P, D, batch count,
digest64 — computed on the device by recon_pipeline_stats) and the
max-over-ranks timing.  The gathered records are identical for every GPU
count (tests/test_shard_gpu.py, tests/test_shard_gloo.py).
"""
from __future__ import annotations

import numpy as np


def shard_range(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous range [g*N/G, (g+1)*N/G) of rank g."""
    return count * rank // world, count * (rank + 1) // world


def run_shard(lib, wl, count: int, world: int, rank: int, chunk: int = 1024, device: int = 0):
    """This rank's shard of the workload's first `count` instances on the
    product library (GPU): returns (start, stats records)."""
    from .pipeline import PipelineRunner
    s, e = shard_range(count, world, rank)
    r = PipelineRunner(lib, wl, max(1, min(chunk, e - s)), device=device)
    return s, r.run_range(s, e - s)


def run_shard_host(lib, wl, count: int, world: int, rank: int):
    """The same through a host-memory library (the CPU checkers): the
    pipeline via recon_pipeline_batch_run_host, the records via
    recon_pipeline_stats over the host outputs."""
    from .inputs import sample_grids
    s, e = shard_range(count, world, rank)
    n = e - s
    occ = sample_grids(wl.seed_base + s, n, wl.W, wl.H, wl.atoms)
    out = lib.pipeline_batch(wl.solver, occ, n, wl.W, wl.H, wl.h_prime, wl.preset, wl.move_stride)
    return s, lib.pipeline_stats_host(out, n, wl.W, wl.h_prime, wl.move_stride)


def gather_to_rank0(dist, arr: np.ndarray, count: int, start: int):
    """Host gather (gloo or nccl object gather) of per-instance arrays,
    concatenated in instance order on rank 0 (None elsewhere)."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (start, arr))
    if dist.get_rank() != 0:
        return None
    full = np.zeros(count, arr.dtype)
    for s, a in parts:
        full[s:s + len(a)] = a
    return full
