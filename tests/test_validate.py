"""On-device validators (recon_validate_batch_run) against the reference's own
validate_solution / check_one_move_per_token / validate_batches.

CPU: the C restatement (oracle) == the compiled reference on valid pipeline
outputs and on seeded corruptions that hit every verdict category.
GPU: the device validators == the oracle on the same cases, then a C3-scale
batch of pipeline outputs validated entirely on the device.
"""
import numpy as np
import pytest

from paper_2504_06182_b200.abi import VERDICT_BITS, verdict_names
from validate_cases import (DAG_EXPLICIT, DAG_NONE, DAG_OCCUPANCY, corruptions, occupancy_edges,
                            pipeline_instances, run, with_dag)

CONFIGS = [  # (solver, W, H, h', atoms, seed, count, preset)
    ("redrec", 32, 32, 16, 614, 1, 4, 0),
    ("bird", 32, 32, 16, 614, 1, 4, 1),
    ("redrec", 24, 20, 9, 260, 77, 4, 1),
    ("bird", 16, 24, 11, 240, 5, 4, 0),
]


def build_cases(lib, per_instance=40, explicit=True):
    rng = np.random.default_rng(0x5EED)
    cases = []
    for cfg in CONFIGS:
        for base in pipeline_instances(lib, *cfg):
            edges = occupancy_edges(lib, base)
            cases.append(("valid", with_dag(base, DAG_OCCUPANCY)))
            for kind, c in corruptions(base, rng, per_instance):
                mode = [DAG_OCCUPANCY, DAG_NONE, DAG_EXPLICIT][int(rng.integers(0, 3 if explicit else 2))]
                if mode == DAG_EXPLICIT:
                    c["_edges"] = edges
                cases.append((f"kind{kind}", with_dag(c, mode, rng, back_edges=int(rng.integers(0, 3)))))
    return cases


@pytest.fixture(scope="module")
def cases(ref):
    return build_cases(ref)


def test_valid_outputs_pass(ref, oracle, cases):
    for name, c in cases:
        if name == "valid":
            assert run(ref, c) == 0 and run(oracle, c) == 0


def test_oracle_matches_reference_on_corruptions(ref, oracle, cases):
    seen = 0
    for name, c in cases:
        vr, vo = run(ref, c), run(oracle, c)
        assert vr == vo, (name, verdict_names(vr), verdict_names(vo))
        assert not (vr & (1 << 31)), (name, verdict_names(vr))
        seen |= vr
    # every category the corruptions can reach shows up
    for bit in ("PATH_BOUNDS", "SHARED_SOURCE", "SHARED_TARGET", "DAG_CYCLE", "STATS_DISPLACEMENT",
                "STATS_DISPLACED", "EXECUTION", "TOKEN_SECOND_PATH", "BATCH_CONSERVATION", "BATCH_BOUND",
                "BATCH_EMPTY", "BATCH_DISJOINT", "BATCH_COLLISION", "BATCH_CONSTRAINT"):
        assert seen & VERDICT_BITS[bit], bit


@pytest.mark.gpu
def test_device_validator_matches_oracle(gpu, oracle, cases):
    for name, c in cases:
        vg, vo = run(gpu, c), run(oracle, c)
        assert vg == vo, (name, verdict_names(vg), verdict_names(vo))


@pytest.mark.gpu
def test_device_validator_on_device_pipeline_c3(gpu, oracle):
    """C3 shape (bird 64x64 h'40 + batching), 256 instances solved and
    batched on the device, validated on the device; a subset cross-checked
    with the oracle."""
    W, H, hp, k, seed, n = 64, 64, 40, 2662, 0x64000000, 256
    for preset in (0, 1):
        insts = pipeline_instances(gpu, "bird", W, H, hp, k, seed, n, preset)
        assert len(insts) > 200
        for c in insts[:8]:
            c = with_dag(c, DAG_OCCUPANCY)
            assert run(gpu, c) == 0 == run(oracle, c)
        # the whole set in one batched call
        P = [len(c["path_src"]) for c in insts]
        D = [len(c["move_batch"]) for c in insts]
        ps, ms = max(P), max(D)
        m = len(insts)
        src = np.zeros(m * ps, np.int32)
        dst = np.zeros(m * ps, np.int32)
        mb = np.zeros(m * ms, np.int32)
        for i, c in enumerate(insts):
            src[i * ps:i * ps + P[i]] = c["path_src"]
            dst[i * ps:i * ps + P[i]] = c["path_dst"]
            mb[i * ms:i * ms + D[i]] = c["move_batch"]
        v = gpu.validate(np.concatenate([c["occ"] for c in insts]), m, W, H, hp, src, dst, ps, np.array(P, np.int32),
                         total_displacement=np.array(D, np.int64), displaced=np.array(P, np.int32),
                         dag_mode=DAG_OCCUPANCY, move_batch=mb, move_stride=ms,
                         batch_count=np.array([c["batch_count"][0] for c in insts], np.int32), preset=preset)
        assert (v == 0).all(), [verdict_names(x) for x in v if x]
        # one corrupted instance in the batch is caught
        mb2 = mb.copy()
        mb2[5 * ms] = mb2[5 * ms] + 1
        v2 = gpu.validate(np.concatenate([c["occ"] for c in insts]), m, W, H, hp, src, dst, ps,
                          np.array(P, np.int32), dag_mode=DAG_OCCUPANCY, move_batch=mb2, move_stride=ms,
                          batch_count=np.array([c["batch_count"][0] for c in insts], np.int32), preset=preset)
        assert v2[5] != 0 and (np.delete(v2, 5) == 0).all()
