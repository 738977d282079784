"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/librecon_ref.so, which
oracle/Makefile compiles from /root/reference/proj/src).  Inputs come from the
reference's own generator contract Rng(seed).sample_without_replacement
(rng.hpp:49-59), reproduced bit-exactly by recon_sample_occ (pinned by
tests/test_inputs.py against the reference's Rng).  The fixtures let the
oracle (CPU) and the B200 path (GPU) be checked on the GPU box, where
/root/reference does not exist.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2504_06182_b200.abi import ReconLib  # noqa: E402
from paper_2504_06182_b200.inputs import sample_chains, sample_grids  # noqa: E402

ref = ReconLib(os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so"), "ref")


def grid_case(name, solver, W, H, hp, k, seed0, count, preset=None):
    occ = sample_grids(seed0, count, W, H, k)
    wpc = (H + 63) // 64
    out = {"occ": occ, "shape": np.array([W, H, hp, k, seed0 & 0xffffffff, count])}
    srcs, dsts, evs, evlog, dags, counts, disps = [], [], [], [], [], [], []
    for i in range(count):
        r = ref.grid_solve(solver, occ[i * W * wpc:(i + 1) * W * wpc], W, H, hp, with_dag=True)
        srcs.append(r.path_src), dsts.append(r.path_dst), evs.append(r.path_event)
        evlog.append(r.events), dags.append(r.dag), counts.append(len(r.path_src))
        disps.append(r.total_displacement)
    out.update(path_src=np.concatenate(srcs), path_dst=np.concatenate(dsts), path_event=np.concatenate(evs),
               events=np.concatenate(evlog), dag=np.concatenate(dags), dag_count=np.array([len(d) for d in dags]),
               path_count=np.array(counts), total_displacement=np.array(disps))
    if preset is not None:
        ms = W * H * 12
        pb = ref.pipeline_batch(solver, occ, count, W, H, hp, preset, ms)
        mb = [pb["move_batch"][i * ms:i * ms + disps[i]] for i in range(count)]
        out.update(preset=np.array([preset]), move_batch=np.concatenate(mb), batch_count=pb["batch_count"],
                   batch_status=pb["status"])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def chain_case(name, n, k, tl, th, seed0, count):
    occ = sample_chains(seed0, count, n, k)
    r = ref.solve_1d_batch(occ, count, n, tl, th)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), occ=occ, shape=np.array([n, k, tl, th, seed0, count]),
                        **r)


if __name__ == "__main__":
    grid_case("c1_redrec", "redrec", 32, 32, 16, 614, 1, 16, preset=0)
    grid_case("c1_bird", "bird", 32, 32, 16, 614, 1, 16, preset=1)
    grid_case("c3_bird", "bird", 64, 64, 40, 2662, 0x64000000, 4, preset=0)
    grid_case("c3_redrec_coldir", "redrec", 64, 64, 40, 2662, 0x64000000, 4, preset=1)
    grid_case("g128_redrec", "redrec", 128, 128, 76, 9830, 0x12800000, 2)
    chain_case("c2_chains", 1024, 563, 256, 767, 0x1D000000, 64)
    grid_case("c3_bird_throw", "bird", 64, 64, 40, 2662, 0x6400001d, 1, preset=0)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
