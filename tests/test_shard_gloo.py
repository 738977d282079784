"""Multi-rank host logic on CPU: world_size 2 over gloo, each rank running its
contiguous shard through a host-memory library behind the same C-ABI (the C
oracle here: this test covers the sharding, the stats records and the
gather; tests/test_shard_gpu.py runs the same on the product library),
gathered on rank 0 and compared with a single-process run: the per-instance
records (digest64 included) must not depend on the rank count."""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ORACLE_LIB
from paper_2504_06182_b200.pipeline import Workload

WL = Workload("small bird+batching 24x24 h'12", "bird", 24, 24, 12, 320, 0x5EED0000, 0, 24 * 24 * 48)
COUNT = 10


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_06182_b200.abi import ReconLib
    from paper_2504_06182_b200.shard import gather_to_rank0, run_shard_host
    lib = ReconLib(ORACLE_LIB, "oracle")
    start, st = run_shard_host(lib, WL, COUNT, world, rank)
    full = gather_to_rank0(dist, st, COUNT, start)
    if rank == 0:
        q.put(full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    from paper_2504_06182_b200.abi import ReconLib
    from paper_2504_06182_b200.shard import run_shard_host, shard_range
    assert [shard_range(10, 2, r) for r in range(2)] == [(0, 5), (5, 10)]
    assert [shard_range(7, 4, r) for r in range(4)] == [(0, 1), (1, 3), (3, 5), (5, 7)]
    lib = ReconLib(ORACLE_LIB, "oracle")
    _, st1 = run_shard_host(lib, WL, COUNT, 1, 0)
    assert (st1["status"] == 0).sum() >= 8 and (st1["batch_count"][st1["status"] == 0] > 0).all()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(full, st1)
