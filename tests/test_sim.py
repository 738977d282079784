"""Multi-cycle loss simulation (recon_sim_run_host; SPEC.md [MODULE] sim).

The reference has no simulation code, so the model is the SPEC's (documented
in include/recon_b200.h).  The checkers run it sequentially on top of their
own solvers (oracle/sim_common.h): the C oracle's, and the compiled
reference's red_rec / bird / batch_moves.  With counter-based draws every
outcome is bit-identical across the three libraries.
"""
import numpy as np
import pytest

from paper_2504_06182_b200.inputs import sample_grids

FIELDS = ("success", "cycles", "status", "n_nu", "n_alpha", "nb_nu", "nb_alpha", "atoms_lost", "elapsed")
LOSSY = dict(p_nu=0.985, p_alpha=0.985, tau=30.0, t_nu=100e-6, t_alpha=300e-6, t_meas=20e-3)


def run(lib, occ, n, W, H, hp, **kw):
    return lib.sim_run(occ, n, W, H, hp, 0xC0FFEE, **kw)


@pytest.mark.parametrize("solver,batching,preset", [("redrec", False, 0), ("bird", True, 0), ("redrec", True, 1)])
def test_checkers_agree(ref, oracle, solver, batching, preset):
    W, H, hp, n = 16, 24, 12, 24
    occ = sample_grids(0x51A0000, n, W, H, int(0.62 * W * H))
    a = run(ref, occ, n, W, H, hp, solver=solver, batching=batching, preset=preset, **LOSSY)
    b = run(oracle, occ, n, W, H, hp, solver=solver, batching=batching, preset=preset, **LOSSY)
    for k in FIELDS:
        assert np.array_equal(a[k], b[k]), k
    assert a["cycles"].max() > 1 and a["atoms_lost"].sum() > 0  # losses matter here


def test_lossless_one_cycle(oracle):
    """SPEC examples: lossless with |S| >= |T| -> success in one cycle; an
    unbatched cycle transfers every displaced token twice."""
    W, H, hp, n = 16, 24, 12, 8
    occ = sample_grids(7, n, W, H, int(0.6 * W * H))
    r = run(oracle, occ, n, W, H, hp, p_nu=1.0, p_alpha=1.0, tau=0.0)
    assert (r["success"] == 1).all() and (r["cycles"] == 1).all() and (r["atoms_lost"] == 0).all()
    assert np.array_equal(r["n_alpha"], 2 * r["nb_alpha"])
    r0 = run(oracle, occ, n, W, H, hp, p_nu=0.0, p_alpha=1.0, tau=0.0, max_cycles=5)
    assert (r0["success"] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("solver,batching,preset", [("redrec", False, 0), ("bird", False, 0), ("bird", True, 0),
                                                    ("redrec", True, 1)])
def test_device_matches_oracle(gpu, oracle, solver, batching, preset):
    W, H, hp, n = 16, 24, 12, 48
    occ = sample_grids(0x51A0000, n, W, H, int(0.62 * W * H))
    a = run(gpu, occ, n, W, H, hp, solver=solver, batching=batching, preset=preset, **LOSSY)
    b = run(oracle, occ, n, W, H, hp, solver=solver, batching=batching, preset=preset, **LOSSY)
    for k in FIELDS:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
def test_device_paper_config(gpu, oracle):
    """SPEC / PAPER §V-C shape: 32x64 grid (W=64 columns here, h'=32 -> a
    32-row band of 64... ) with the paper's loss probabilities; device ==
    oracle on a subset, success probability in (0, 1)."""
    W, H, hp, n = 64, 32, 16, 64
    occ = sample_grids(0x0A0B0000, n, W, H, int(0.6 * W * H))
    kw = dict(solver="bird", batching=False, **LOSSY)
    a = run(gpu, occ, n, W, H, hp, **kw)
    b = run(oracle, occ[: 8 * W], 8, W, H, hp, **kw)
    for k in FIELDS:
        assert np.array_equal(a[k][:8], b[k]), k
    assert 0 < a["success"].mean() < 1


def test_batching_conservation(oracle):
    """SPEC invariant: N_nu and N_alpha are identical with and without
    batching on the same trial seed; only NB counts and elapsed time differ.
    (Without lifetime decay: decay depends on the elapsed time, which batching
    changes.)"""
    W, H, hp, n = 16, 24, 12, 16
    occ = sample_grids(0x51A0000, n, W, H, int(0.62 * W * H))
    kw = dict(LOSSY, tau=0.0)
    a = run(oracle, occ, n, W, H, hp, solver="bird", batching=False, **kw)
    b = run(oracle, occ, n, W, H, hp, solver="bird", batching=True, preset=0, **kw)
    for k in ("success", "cycles", "n_nu", "n_alpha", "atoms_lost"):
        assert np.array_equal(a[k], b[k]), k
    assert (b["nb_nu"] < a["nb_nu"]).all() and (b["elapsed"] < a["elapsed"]).all()
