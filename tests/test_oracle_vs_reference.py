"""Pins the C restatement (oracle/recon_oracle.c) against the compiled
reference (oracle/_ref) on randomized instances: red-rec, bird, DAG, event
logs, chains, generalized assignment, batching (both presets)."""
import numpy as np
import pytest

from helpers import call, random_band_instance, same_grid


@pytest.mark.parametrize("solver", ["redrec", "bird"])
def test_grid_random(oracle, ref, solver):
    rng = np.random.default_rng(0xa11ce)
    for it in range(800):
        occ, W, H, hp = random_band_instance(rng, 16, 24, critical=bool(it % 2))
        (o, eo), (r, er) = call(oracle, "grid_solve", solver, occ, W, H, hp, with_dag=True), \
            call(ref, "grid_solve", solver, occ, W, H, hp, with_dag=True)
        assert eo == er, it
        if r is not None:
            assert same_grid(o, r), (it, W, H, hp)


@pytest.mark.parametrize("solver", ["redrec", "bird"])
def test_grid_medium(oracle, ref, solver):
    rng = np.random.default_rng(0xbee)
    for it in range(30):
        occ, W, H, hp = random_band_instance(rng, 80, 100, critical=bool(it % 2))
        o = oracle.grid_solve(solver, occ, W, H, hp, with_dag=True)
        r = ref.grid_solve(solver, occ, W, H, hp, with_dag=True)
        assert same_grid(o, r), it


def test_chains_random(oracle, ref):
    rng = np.random.default_rng(0xc4a1)
    for it in range(1500):
        n = int(rng.integers(1, 80))
        ns = int(rng.integers(0, n + 1))
        nt = int(rng.integers(0, ns + 1)) if ns else 0
        S = rng.choice(n, ns, replace=False)
        T = rng.choice(n, nt, replace=False)
        (o, eo), (r, er) = call(oracle, "solve_1d", n, S, T), call(ref, "solve_1d", n, S, T)
        assert eo == er
        if r is not None:
            for key in ("path_src", "path_dst", "path_order", "dag"):
                assert np.array_equal(getattr(o, key), getattr(r, key)), (it, key)


def test_generalized_random(oracle, ref):
    rng = np.random.default_rng(0x9e2)
    for it in range(1500):
        np_ = int(rng.integers(1, 6))
        pos = np.sort(rng.choice(np.arange(-6, 20), np_, replace=False))
        mult = rng.integers(1, 4, np_)
        mu = np.array([rng.integers(0, m + 1) for m in mult])
        tg = np.sort(rng.choice(np.arange(-6, 20), int(rng.integers(0, 7)), replace=False))
        (o, eo), (r, er) = call(oracle, "assign_1d_generalized", pos, mult, mu, tg), \
            call(ref, "assign_1d_generalized", pos, mult, mu, tg)
        assert eo == er
        if r is not None:
            assert o[0] == r[0] and np.array_equal(o[1], r[1]) and np.array_equal(o[2], r[2])


@pytest.mark.parametrize("preset", [0, 1])
def test_pipeline_random(oracle, ref, preset):
    rng = np.random.default_rng(0x7e57 + preset)
    for it in range(150):
        occ, W, H, hp = random_band_instance(rng, 24, 32, critical=bool(it % 2))
        for solver in ("redrec", "bird"):
            ms = W * H * (W + H)
            o = oracle.pipeline_batch(solver, occ, 1, W, H, hp, preset, ms)
            r = ref.pipeline_batch(solver, occ, 1, W, H, hp, preset, ms)
            assert np.array_equal(o["status"], r["status"])
            if r["status"][0] == 0:
                d = int(r["total_displacement"][0])
                assert o["batch_count"][0] == r["batch_count"][0]
                assert np.array_equal(o["move_batch"][:d], r["move_batch"][:d])


@pytest.mark.parametrize("solver", ["redrec", "bird"])
def test_packed_batch_format(oracle, ref, solver):
    """*_batch_host_packed (src | dst << 16 per path) in both CPU libraries
    against the unpacked batch call; grids over 65,536 cells are refused."""
    from paper_2504_06182_b200.inputs import sample_grids
    W, H, hp, n = 24, 20, 10, 12
    occ = sample_grids(0x9ac, n, W, H, 300)
    r = ref.grid_solve_batch(solver, occ, n, W, H, hp)
    for lib in (oracle, ref):
        p = lib.grid_solve_batch_packed(solver, occ, n, W, H, hp)
        for key in ("path_count", "total_displacement", "status"):
            assert np.array_equal(p[key], r[key]), key
        S = W * hp
        for i in range(n):
            c = int(r["path_count"][i])
            pk = p["path_packed"][i * S:i * S + c]
            assert np.array_equal((pk & 0xFFFF).astype(np.int32), r["path_src"][i * S:i * S + c])
            assert np.array_equal((pk >> 16).astype(np.int32), r["path_dst"][i * S:i * S + c])
        with pytest.raises(Exception):
            lib.grid_solve_batch_packed(solver, sample_grids(1, 1, 300, 300, 50000), 1, 300, 300, 100)
