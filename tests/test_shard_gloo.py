"""Multi-rank path on CPU: world_size 2 over gloo, each rank solving its
contiguous shard (here with the C oracle standing in for the GPU, since the
test covers the host-side sharding and gather logic), gathered on rank 0 and
compared with a single-process run: outputs must not depend on the rank count."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ORACLE_LIB

W, H, HP, K, SEED, COUNT = 24, 24, 12, 320, 0x5EED0000, 10


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_06182_b200.abi import ReconLib
    from paper_2504_06182_b200.shard import gather_to_rank0, solve_shard
    lib = ReconLib(ORACLE_LIB, "oracle")
    start, dig, td = solve_shard(lib, "redrec", SEED, COUNT, W, H, HP, K, world, rank)
    full_d = gather_to_rank0(dist, dig, COUNT, start)
    full_t = gather_to_rank0(dist, td, COUNT, start)
    if rank == 0:
        q.put((full_d, full_t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    from paper_2504_06182_b200.abi import ReconLib
    from paper_2504_06182_b200.shard import shard_range, solve_shard
    assert [shard_range(10, 2, r) for r in range(2)] == [(0, 5), (5, 10)]
    assert [shard_range(7, 4, r) for r in range(4)] == [(0, 1), (1, 3), (3, 5), (5, 7)]
    lib = ReconLib(ORACLE_LIB, "oracle")
    _, dig1, td1 = solve_shard(lib, "redrec", SEED, COUNT, W, H, HP, K, 1, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full_d, full_t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(full_d, dig1)
    assert np.array_equal(full_t, td1)
