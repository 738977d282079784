"""GPU parity of red-rec and bird (recon_redrec_solve / recon_bird_solve)
against the C oracle and the compiled reference: bit-exact path list in
canonical order, event log, stats and occupancy DAG."""
import numpy as np
import pytest

from helpers import call, random_band_instance, same_grid
from paper_2504_06182_b200.inputs import grid_from_depths, sample_grids

pytestmark = pytest.mark.gpu

SOLVERS = ("redrec", "bird")


@pytest.mark.parametrize("solver", SOLVERS)
def test_random_small_instances_match_oracle(gpu, oracle, solver):
    rng = np.random.default_rng(0x5ed5ec)
    bad = []
    for it in range(400):
        occ, W, H, hp = random_band_instance(rng, 16, 24, critical=bool(it % 2))
        (g, eg), (o, eo) = call(gpu, "grid_solve", solver, occ, W, H, hp, with_dag=True), \
            call(oracle, "grid_solve", solver, occ, W, H, hp, with_dag=True)
        if eg or eo:
            if eg != eo:
                bad.append((it, eg, eo))
            continue
        if not same_grid(g, o):
            bad.append((it, W, H, hp))
    assert not bad, bad[:5]


@pytest.mark.parametrize("solver", SOLVERS)
def test_random_medium_instances_match_reference(gpu, ref, solver):
    rng = np.random.default_rng(0xb16b16)
    bad = []
    for it in range(60):
        occ, W, H, hp = random_band_instance(rng, 96, 130, critical=bool(it % 2))
        (g, eg), (r, er) = call(gpu, "grid_solve", solver, occ, W, H, hp, with_dag=True), \
            call(ref, "grid_solve", solver, occ, W, H, hp, with_dag=True)
        if eg or er:
            if eg != er:
                bad.append((it, eg, er))
            continue
        if not same_grid(g, r):
            bad.append((it, W, H, hp))
    assert not bad, bad[:5]


@pytest.mark.parametrize("solver", SOLVERS)
def test_pinned_reference_flows(gpu, solver):
    # test_redrec.cpp:236-349 / test_bird.cpp:156-262 pinned displacements
    cases = {
        "redrec": [((4, 6, 2, [[0, 2, 3], [2, 3], [2, 3], [2]]), 6, 2),
                   ((3, 6, 2, [[1, 2, 3], [], [1, 2, 3]]), 5, 2),
                   ((2, 6, 2, [[2, 3, 5], [0]]), 5, 2),
                   ((3, 9, 3, [[0, 2, 3, 4, 5], [4], [0, 2, 3, 4, 5]]), 8, None)],
        "bird": [((3, 5, 1, [[], [2], [1, 2]]), 3, None),
                 ((5, 6, 2, [[2, 3], [1, 2, 3], [], [1, 2, 3], [2, 3]]), 5, None),
                 ((6, 12, 2, [[5, 6], [5, 6], [], [2, 5, 6], [5, 6], [4, 5, 6]]), 9, 2),
                 ((2, 12, 2, [[0], [3, 4, 5, 6]]), 6, 2),
                 ((3, 6, 2, [[5], [0], [0, 1, 2, 3]]), 11, None),
                 ((3, 9, 3, [[0, 2, 3, 4, 5], [4], [0, 2, 3, 4, 5]]), 6, None),
                 ((1, 5, 2, [[0, 2, 4]]), 1, 1),
                 ((5, 4, 1, [[0, 2], [], [2], [], [0, 2]]), 6, None)],
    }[solver]
    for (W, H, hp, depths), disp, npaths in cases:
        g = gpu.grid_solve(solver, grid_from_depths(depths, H), W, H, hp)
        assert g.total_displacement == disp
        if npaths is not None:
            assert len(g.path_src) == npaths
    if solver == "bird":
        g = gpu.grid_solve("bird", grid_from_depths([[5], [0], [0, 1, 2, 3]], 6), 3, 6, 2)
        assert list(g.events) == [2, 0, 1]
        g = gpu.grid_solve("bird", grid_from_depths([[0, 2], [], [2], [], [0, 2]], 4), 5, 4, 1)
        assert list(g.events) == [0, 2, 4, 1, 3]


@pytest.mark.parametrize("solver,W,H,hp,k,seed0,n", [
    ("redrec", 32, 32, 16, 614, 1, 40),         # C1
    ("bird", 64, 64, 40, 2662, 0x64000000, 12),  # C3 shape
    ("redrec", 64, 64, 40, 2662, 0x64000000, 12),
])
def test_seeded_configs_match_reference(gpu, ref, solver, W, H, hp, k, seed0, n):
    occ = sample_grids(seed0, n, W, H, k)
    wpc = (H + 63) // 64
    for i in range(n):
        o = occ[i * W * wpc:(i + 1) * W * wpc]
        g = gpu.grid_solve(solver, o, W, H, hp, with_dag=True)
        r = ref.grid_solve(solver, o, W, H, hp, with_dag=True)
        assert same_grid(g, r), (solver, i)


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("hp,seed", [(128, 256), (153, 257)])
def test_c4_256_matches_reference(gpu, ref, solver, hp, seed):
    occ = sample_grids(seed, 1, 256, 256, 39322)
    g = gpu.grid_solve(solver, occ, 256, 256, hp, with_dag=True)
    r = ref.grid_solve(solver, occ, 256, 256, hp, with_dag=True)
    assert same_grid(g, r)


@pytest.mark.parametrize("solver", SOLVERS)
def test_batched_host_api_matches_single(gpu, oracle, solver):
    W, H, hp, k, n = 48, 40, 24, 1200, 64
    occ = sample_grids(0xC0FFEE, n, W, H, k)
    out = gpu.grid_solve_batch(solver, occ, n, W, H, hp)
    ora = oracle.grid_solve_batch(solver, occ, n, W, H, hp)
    for key in ("path_count", "total_displacement", "status", "events"):
        assert np.array_equal(out[key], ora[key]), key
    stride = W * hp
    for i in range(n):
        c = out["path_count"][i]
        for key in ("path_src", "path_dst", "path_event"):
            assert np.array_equal(out[key][i * stride:i * stride + c], ora[key][i * stride:i * stride + c])


@pytest.mark.parametrize("solver", SOLVERS)
def test_error_statuses(gpu, solver):
    from paper_2504_06182_b200.abi import InfeasibleError, InputError
    occ = grid_from_depths([[1], [2]], 4)
    with pytest.raises(InfeasibleError):
        gpu.grid_solve(solver, occ, 2, 4, 2)
    with pytest.raises(InputError):
        gpu.grid_solve(solver, occ, 2, 4, 4)
    with pytest.raises(InputError):
        gpu.grid_solve(solver, occ, 2, 4, 0)


@pytest.mark.parametrize("solver", SOLVERS)
def test_c4_batch_of_256_matches_reference(gpu, ref, solver):
    """More instances than SMs: the 4-warp batch CTAs (and, for red-rec, the
    planner kernel + executor on many instances at once), against the compiled
    reference on every instance."""
    W = H = 256
    n = 160
    occ = sample_grids(0x25600000, n, W, H, 39322)
    g = gpu.grid_solve_batch(solver, occ, n, W, H, 153)
    r = ref.grid_solve_batch(solver, occ, n, W, H, 153)
    for key in ("path_count", "total_displacement", "status"):
        assert np.array_equal(g[key], r[key]), key
    S = W * 153
    for i in range(n):
        P = int(r["path_count"][i])
        for key in ("path_src", "path_dst"):
            assert np.array_equal(g[key][i * S:i * S + P], r[key][i * S:i * S + P]), (key, i)


@pytest.mark.parametrize("solver", SOLVERS)
def test_more_instances_than_ctas_matches_reference(gpu, ref, solver):
    """More instances than resident CTAs (2-warp CTAs at 128^2): CTAs claim
    further instances from the global counter (dynamic scheduling)."""
    W = H = 128
    n = 3000
    occ = sample_grids(0x12800000, n, W, H, 9830)
    g = gpu.grid_solve_batch(solver, occ, n, W, H, 77)
    r = ref.grid_solve_batch(solver, occ, n, W, H, 77)
    for key in ("path_count", "total_displacement", "status"):
        assert np.array_equal(g[key], r[key]), key
    S = W * 77
    for i in range(n):
        P = int(r["path_count"][i])
        for key in ("path_src", "path_dst"):
            assert np.array_equal(g[key][i * S:i * S + P], r[key][i * S:i * S + P]), (key, i)


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("W,hp,n,k,seed", [(256, 153, 160, 39322, 0x25600000), (128, 77, 3000, 9830, 0x12800000)])
def test_packed_host_api_matches_reference(gpu, ref, solver, W, hp, n, k, seed):
    """*_batch_host_packed (src | dst << 16 per path, several copy chunks at
    128^2) against the compiled reference on every instance."""
    occ = sample_grids(seed, n, W, W, k)
    g = gpu.grid_solve_batch_packed(solver, occ, n, W, W, hp)
    r = ref.grid_solve_batch(solver, occ, n, W, W, hp)
    for key in ("path_count", "total_displacement", "status"):
        assert np.array_equal(g[key], r[key]), key
    S = W * hp
    for i in range(n):
        P = int(r["path_count"][i])
        pk = g["path_packed"][i * S:i * S + P]
        assert np.array_equal((pk & 0xFFFF).astype(np.int32), r["path_src"][i * S:i * S + P]), ("src", i)
        assert np.array_equal((pk >> 16).astype(np.int32), r["path_dst"][i * S:i * S + P]), ("dst", i)


def test_packed_host_api_rejects_large_grids(gpu):
    occ = sample_grids(1, 1, 512, 512, 157286)
    with pytest.raises(Exception):
        gpu.grid_solve_batch_packed("redrec", occ, 1, 512, 512, 307)


@pytest.mark.parametrize("solver", SOLVERS)
def test_c5_512_matches_reference(gpu, ref, solver):
    occ = sample_grids(0x51200000, 1, 512, 512, 157286)
    g = gpu.grid_solve(solver, occ, 512, 512, 307, with_dag=True)
    r = ref.grid_solve(solver, occ, 512, 512, 307, with_dag=True)
    assert same_grid(g, r)


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("W,H,hp,eps", [(1000, 8, 3, 0.5), (4, 1000, 500, 0.55), (1024, 64, 40, 0.66),
                                         (96, 1024, 600, 0.62)])
def test_extreme_shapes_match_oracle(gpu, oracle, solver, W, H, hp, eps):
    occ = sample_grids(0xE57, 2, W, H, int(round(eps * W * H)))
    wpc = (H + 63) // 64
    for i in range(2):
        o = occ[i * W * wpc:(i + 1) * W * wpc]
        (g, eg), (r, er) = call(gpu, "grid_solve", solver, o, W, H, hp), call(oracle, "grid_solve", solver, o, W, H, hp)
        assert eg == er
        if g is not None:
            assert same_grid(g, r)
