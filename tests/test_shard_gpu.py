"""Multi-rank path on the PRODUCT library: two ranks over
gloo, both on the one GPU of the box (the timing of such a run means nothing;
the outputs do), each running its contiguous shard of C5 (bird + batching
512^2) and C3 through pipeline.PipelineRunner, the per-instance stats records
(device digest64) gathered on rank 0.  They must equal a single-process run
and the reference's fixtures (tests/golden/scale_*.npz)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu
JOBS = (("c5", 16), ("c3", 512))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_06182_b200 import load_native
    from paper_2504_06182_b200.pipeline import C3, C5
    from paper_2504_06182_b200.shard import gather_to_rank0, run_shard
    lib = load_native()
    res = {}
    for name, count in JOBS:
        start, st = run_shard(lib, {"c5": C5, "c3": C3}[name], count, world, rank)
        res[name] = gather_to_rank0(dist, st, count, start)
    if rank == 0:
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_product_matches_single_rank_and_reference(gpu):
    from paper_2504_06182_b200.pipeline import C3, C5
    from paper_2504_06182_b200.shard import run_shard
    single = {name: run_shard(gpu, {"c5": C5, "c3": C3}[name], count, 1, 0)[1] for name, count in JOBS}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, count in JOBS:
        assert np.array_equal(res[name], single[name]), name
        g = np.load(os.path.join(ROOT, "tests", "golden", f"scale_{name}_none.npz"))
        assert np.array_equal(res[name]["digest"], g["digest"][:count]), name
        assert np.array_equal(res[name]["status"], g["status"][:count]), name
