"""Multi-GPU sharding of independent instances.

Instances are independent pure functions of their seed, so a batch is split
into contiguous per-rank ranges and every rank solves its range on its own
GPU; there is no collective on the data path.  torch.distributed only
carries the final host gather of per-instance results (digests + stats) and
the max-over-ranks timing.
"""
from __future__ import annotations

import hashlib

import numpy as np


def shard_range(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous range [g*N/G, (g+1)*N/G) of rank g."""
    return count * rank // world, count * (rank + 1) // world


def instance_digests(out: dict, count: int, stride: int) -> np.ndarray:
    """64-bit digest of each instance's canonical path list (+ status)."""
    d = np.zeros(count, np.uint64)
    for i in range(count):
        c = int(out["path_count"][i])
        h = hashlib.blake2b(digest_size=8)
        h.update(np.int32(out["status"][i]).tobytes())
        h.update(out["path_src"][i * stride:i * stride + c].tobytes())
        h.update(out["path_dst"][i * stride:i * stride + c].tobytes())
        d[i] = np.frombuffer(h.digest(), np.uint64)[0]
    return d


def solve_shard(lib, solver: str, seed_base: int, count: int, W: int, H: int, hp: int, k: int,
                world: int, rank: int):
    """Solves this rank's shard of `count` seeded instances; returns (start, digests, total displacement)."""
    from .inputs import sample_grids
    s, e = shard_range(count, world, rank)
    occ = sample_grids(seed_base + s, e - s, W, H, k)
    out = lib.grid_solve_batch(solver, occ, e - s, W, H, hp, host=True, with_events=False)
    return s, instance_digests(out, e - s, W * hp), out["total_displacement"].copy()


def gather_to_rank0(dist, arr: np.ndarray, count: int, start: int):
    """Host gather (gloo or nccl object gather) of per-instance arrays, concatenated in instance order."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (start, arr))
    if dist.get_rank() != 0:
        return None
    full = np.zeros(count, arr.dtype)
    for s, a in parts:
        full[s:s + len(a)] = a
    return full
