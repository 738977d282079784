"""Batching parity at C3 / C4 / C5 scale.

Every instance's status, batch count and digest64 (paths + the whole batch
schedule, include/recon_b200.h; tests/digest.py) are compared with fixtures
generated from the UNMODIFIED reference (oracle/_ref, tests/golden/
make_batch_scale.py), and a few instances are compared in full against the
compiled reference run live on this host.  Every kernel variant of the
pipeline batching (batching.cu / batch_wide.cu) is forced at least once on
the grids that select it by default only at scale.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from digest import pipeline_digests
from paper_2504_06182_b200.abi import expand_runs
from paper_2504_06182_b200.inputs import sample_grids
from paper_2504_06182_b200.pipeline import C3, C4, C5, PipelineRunner

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(ROOT, "tests", "golden")

# bird / preset none throws "batching made no progress"
# (batching.cpp:127-128) on exactly these 21 of the 4,096 C3 seeds
C3_THROWS = [0x6400001d, 0x640000b0, 0x64000236, 0x64000357, 0x640003ca, 0x64000422, 0x64000487, 0x640004bc,
             0x64000546, 0x6400064b, 0x64000681, 0x64000781, 0x64000866, 0x64000919, 0x640009ae, 0x64000aaf,
             0x64000b55, 0x64000c5c, 0x64000d02, 0x64000eae, 0x64000f17]


def golden(name):
    return np.load(os.path.join(GOLDEN, f"scale_{name}.npz"))


def check(stats, g, first=0):
    n = len(stats)
    assert np.array_equal(stats["status"], g["status"][first:first + n])
    ok = stats["status"] == 0
    assert np.array_equal(stats["batch_count"][ok], g["batch_count"][first:first + n][ok].astype(np.int64))
    assert np.array_equal(stats["total_displacement"][ok], g["total_displacement"][first:first + n][ok])
    bad = np.nonzero(stats["digest"] != g["digest"][first:first + n])[0]
    assert len(bad) == 0, f"digest mismatch at instances {bad[:10] + first}"


def variant(env, name, first, count, preset=None):
    e = dict(os.environ)
    e.update(env)
    cmd = [sys.executable, os.path.join(ROOT, "tests", "scale_variant.py"), name, str(first), str(count)]
    if preset is not None:
        cmd.append(str(preset))
    r = subprocess.run(cmd, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    st = np.zeros(count, [("status", np.int32), ("batch_count", np.int64), ("total_displacement", np.int64),
                          ("digest", np.uint64)])
    st["status"] = d["status"]
    st["batch_count"] = d["batch_count"]
    st["digest"] = [int(x) for x in d["digest"]]
    return st


def check_variant(st, g, first=0):
    n = len(st)
    assert np.array_equal(st["status"], g["status"][first:first + n])
    ok = st["status"] == 0
    assert np.array_equal(st["batch_count"][ok], g["batch_count"][first:first + n][ok].astype(np.int64))
    assert np.array_equal(st["digest"], g["digest"][first:first + n])


@pytest.fixture(scope="module")
def runner_c3(gpu):
    return PipelineRunner(gpu, C3, 4096)


def test_c3_all_4096_none(runner_c3):
    st = runner_c3.run_range(0, 4096)
    check(st, golden("c3_none"))
    throws = sorted(C3.seed_base + int(i) for i in np.nonzero(st["status"] != 0)[0])
    assert throws == C3_THROWS
    assert (st["status"][st["status"] != 0] == 1).all()  # InputError
    assert (st["detail"][st["status"] != 0] != 0).all()


def test_c3_all_4096_column_direction(gpu):
    r = PipelineRunner(gpu, C3, 4096, preset=1)
    check(r.run_range(0, 4096), golden("c3_coldir"))


@pytest.mark.parametrize("preset,name", [(0, "c4_none"), (1, "c4_coldir")])
def test_c4_redrec_h153(gpu, preset, name):
    r = PipelineRunner(gpu, C4, 8, preset=preset)
    check(r.run_range(0, 8), golden(name))


def test_c5_64_none(gpu):
    r = PipelineRunner(gpu, C5, 64)
    st = r.run_range(0, 64)
    check(st, golden("c5_none"))
    # seeds 0x51200009, ... end in the no-progress throw after ~1.8 M batches
    assert (st["status"] != 0).any() and (st["status"] == 0).sum() >= 48


def test_c5_full_outputs_vs_live_reference(gpu, ref):
    """Two C5 instances (one completes, one ends in the no-progress throw),
    every path and every move's batch index against the compiled reference."""
    r = PipelineRunner(gpu, C5, 2)
    occ = np.concatenate([sample_grids(C5.seed_base + i, 1, 512, 512, C5.atoms) for i in (0, 9)])
    r.load(occ, 2)
    r.run(2)
    stats = r.stats(2)
    g = r.outputs()
    o = ref.pipeline_batch("bird", occ, 2, 512, 512, 307, 0, C5.move_stride)
    assert np.array_equal(g["status"], o["status"]) and list(o["status"]) == [0, 1]
    assert g["batch_count"][0] == o["batch_count"][0] == 1879785
    P, D = int(o["path_count"][0]), int(o["total_displacement"][0])
    assert np.array_equal(g["path_src"][:P], o["path_src"][:P])
    assert np.array_equal(g["path_dst"][:P], o["path_dst"][:P])
    assert np.array_equal(g["move_batch"][:D], o["move_batch"][:D])
    # the device digest is tests/digest.py's and the checkers' recon_pipeline_stats
    d_np = pipeline_digests(o, 2, C5.paths, C5.move_stride)
    assert np.array_equal(stats["digest"], d_np)
    assert np.array_equal(ref.pipeline_stats_host(o, 2, 512, 307, C5.move_stride)["digest"], d_np)
    # the run-length schedule of the host call expands to the reference's schedule
    rr = gpu.pipeline_batch_runs("bird", occ, 2, 512, 512, 307, 0, C5.move_stride)
    assert int(rr["run_count"][0]) < P + 10_000 and int(rr["run_count"][1]) == 0
    assert np.array_equal(expand_runs(rr["run_slot"], rr["run_batch"], int(rr["run_count"][0]), D), o["move_batch"][:D])


def test_schedule_runs_device_equals_oracle(gpu, oracle):
    """recon_pipeline_batch_run_host_runs on the device == the C oracle's, run
    for run, on 256 C3 instances (both presets) and 4 C4 instances (none; the
    oracle's column_direction C4 takes ~1 M batches per instance)."""
    for wl, n, presets in ((C3, 256, (0, 1)), (C4, 4, (0,))):
        occ = sample_grids(wl.seed_base, n, wl.W, wl.H, wl.atoms)
        for preset in presets:
            g = gpu.pipeline_batch_runs(wl.solver, occ, n, wl.W, wl.H, wl.h_prime, preset, wl.move_stride)
            o = oracle.pipeline_batch_runs(wl.solver, occ, n, wl.W, wl.H, wl.h_prime, preset, wl.move_stride)
            assert np.array_equal(g["run_count"], o["run_count"]) and np.array_equal(g["status"], o["status"])
            if wl is C3 and preset == 0:  # page-locked run arrays: written by runs_to_host_kernel, not copied
                p = gpu.pipeline_batch_runs(wl.solver, occ, n, wl.W, wl.H, wl.h_prime, preset, wl.move_stride,
                                            pinned=True)
                assert np.array_equal(p["run_count"], g["run_count"])
                assert np.array_equal(p["run_slot"], g["run_slot"]) and np.array_equal(p["run_batch"], g["run_batch"])
            rs = g["run_stride"]
            for i in range(n):
                k = int(g["run_count"][i])
                assert np.array_equal(g["run_slot"][i * rs:i * rs + k], o["run_slot"][i * rs:i * rs + k])
                assert np.array_equal(g["run_batch"][i * rs:i * rs + k], o["run_batch"][i * rs:i * rs + k])


def test_device_stats_record(gpu, oracle):
    """recon_pipeline_stats: device == oracle == tests/digest.py, and the
    SolutionStats fields, on 64 C3 instances (incl. a throwing one)."""
    r = PipelineRunner(gpu, C3, 64)
    occ = sample_grids(C3.seed_base, 64, 64, 64, C3.atoms)
    r.load(occ, 64)
    r.run(64)
    st = r.stats(64)
    out = r.outputs()
    o = oracle.pipeline_batch("bird", occ, 64, 64, 64, 40, 0, C3.move_stride)
    so = oracle.pipeline_stats_host(o, 64, 64, 40, C3.move_stride)
    assert np.array_equal(st, so)
    assert np.array_equal(st["digest"], pipeline_digests(out, 64, C3.paths, C3.move_stride))
    ok = st["status"] == 0
    assert np.array_equal(st["displaced_tokens"][ok], st["path_count"][ok])  # solvers emit no empty path
    assert st["status"][0x1d] == 1


# ---- forced kernel variants (each selected by default only at scale) ----------

@pytest.mark.parametrize("env", [
    {"RECON_BATCH_LEAP": "0"},                                  # batch-by-batch warp loop (modes 1/9 at >148 instances)
    {"RECON_BATCH_LEAP": "0", "RECON_BATCH_OCC_SMEM": "0"},     # mode 0: bitmaps in global memory
    {"RECON_BATCH_WIDE": "0"},                                  # leap without the wide phase (general warp path)
    {"RECON_WIDE_SMEM_KB": "105"},                              # wide ready set outgrows shared memory mid-run
    {"RECON_WIDE_SMEM_KB": "80"},                               # windows halved by overflowing plans
    {"RECON_WIDE_SMEM_KB": "60"},                               # ... or at batch 0 (warp kernel from scratch)
    {"RECON_WIDE_WINDOW": "0"},                                 # the wide phase batch by batch (batch_wide.cu)
    {"RECON_WIDE_WINDOW": "0", "RECON_WIDE_SMEM_KB": "105"},
])
def test_c5_variants(env):
    # 160 instances > 148 SMs: the many-instance shapes (4-warp batch CTAs,
    # occupancy-only shared memory) are the ones C5 selects
    st = variant(env, "c5", 0, 160 if env.get("RECON_BATCH_LEAP") == "0" and len(env) == 1 else 8)
    check_variant(st, golden("c5_none"))


@pytest.mark.parametrize("env", [
    {"RECON_BATCH_WIDE": "0"},
    {"RECON_WIDE_WINDOW": "0"},
    {"RECON_WALK_LANES": "32"},                                 # the DAG walk with a warp per path
    {"RECON_WALK_LANES": "16"},
    {"RECON_BATCH_LEAP": "0", "RECON_BATCH_BSM": "0"},
    {"RECON_BATCH_LEAP": "0", "RECON_BATCH_WIDE": "0", "RECON_BATCH_LOG": "1"},
])
def test_c4_variants(env):
    check_variant(variant(env, "c4", 0, 8), golden("c4_none"))


@pytest.mark.parametrize("env", [
    {"RECON_BATCH_LEAP": "2"},                                  # leap mode on small grids (shared-memory bitmaps)
    {"RECON_BATCH_LEAP": "0", "RECON_BATCH_LOG": "0", "RECON_BATCH_BSM": "0"},
    {"RECON_BATCH_WIDE": "1"},
    {"RECON_BATCH_WIDE": "1", "RECON_WIDE_WINDOW": "0"},
    {"RECON_BATCH_WIDE": "1", "RECON_BATCH_LEAP": "2"},
    {"RECON_SMALL_DAG": "0"},
    {"RECON_SMALL_DAG": "0", "RECON_WALK_LANES": "32"},
    {"RECON_SMALL_DAG": "0", "RECON_WALK_LANES": "1"},
])
def test_c3_variants(env):
    check_variant(variant(env, "c3", 0, 4096), golden("c3_none"))
