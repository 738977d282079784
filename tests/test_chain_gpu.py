"""GPU parity of the exact-1D path (recon_assign_1d / recon_assign_1d_generalized /
recon_solve_1d / recon_solve_1d_batch) against the compiled reference."""
import numpy as np
import pytest

from helpers import call
from paper_2504_06182_b200.inputs import sample_chains

pytestmark = pytest.mark.gpu


def _same_chain(a, b):
    return (np.array_equal(a.path_src, b.path_src) and np.array_equal(a.path_dst, b.path_dst)
            and np.array_equal(a.path_order, b.path_order) and np.array_equal(a.dag, b.dag)
            and a.total_displacement == b.total_displacement and a.displaced == b.displaced)


def _random_chain(rng, max_n, band=False):
    n = int(rng.integers(1, max_n + 1))
    ns = int(rng.integers(0, n + 1))
    nt = int(rng.integers(0, ns + 1)) if ns else 0
    S = rng.choice(n, ns, replace=False)
    if band and nt:
        lo = int(rng.integers(0, n - nt + 1))
        T = np.arange(lo, lo + nt)
    else:
        T = rng.choice(n, nt, replace=False)
    return n, S, T


@pytest.mark.parametrize("band", [False, True])
def test_solve_1d_random_matches_reference(gpu, ref, band):
    rng = np.random.default_rng(0x501e + band)
    bad = []
    for it in range(500):
        n, S, T = _random_chain(rng, 40 if not band else 300, band)
        (g, eg), (r, er) = call(gpu, "solve_1d", n, S, T), call(ref, "solve_1d", n, S, T)
        if eg or er:
            if eg != er:
                bad.append((it, eg, er))
            continue
        if not _same_chain(g, r):
            bad.append((it, n, list(S), list(T)))
    assert not bad, bad[:3]


@pytest.mark.parametrize("band", [False, True])
def test_assign_1d_random_matches_reference(gpu, ref, band):
    rng = np.random.default_rng(0x1d5eed + band)
    bad = []
    for it in range(500):
        n, S, T = _random_chain(rng, 60, band)
        (g, eg), (r, er) = call(gpu, "assign_1d", n, S, T), call(ref, "assign_1d", n, S, T)
        if eg or er:
            if eg != er:
                bad.append((it, eg, er))
            continue
        if not (g[0] == r[0] and np.array_equal(g[1], r[1]) and np.array_equal(g[2], r[2])):
            bad.append((it, n, list(S), list(T)))
    assert not bad, bad[:3]


def test_assign_1d_errors(gpu):
    from paper_2504_06182_b200.abi import InfeasibleError, InputError
    # test_exact1d.cpp:76-83
    with pytest.raises(InfeasibleError):
        gpu.assign_1d(4, [0], [1, 2])
    for args in ((4, [0, 4], [1]), (4, [-1, 2], [1]), (4, [2, 2], [1]), (4, [0, 2], [1, 1]), (0, [], [])):
        with pytest.raises(InputError):
            gpu.assign_1d(*args)


def test_assign_1d_pinned(gpu):
    w, pairs, use = gpu.assign_1d(6, [0, 2, 5], [1, 2, 3])  # test_exact1d.cpp:51-60
    assert w == 3 and pairs.tolist() == [[0, 1], [2, 2], [5, 3]] and use.tolist() == [1, 1, 1]
    w, pairs, use = gpu.assign_1d(5, [0, 1, 4], [2])  # :68-74
    assert w == 1 and pairs.tolist() == [[1, 2]] and use.tolist() == [0, 1, 0]
    w, pairs, _ = gpu.assign_1d(6, [0, 1, 5], [2, 3])  # :92-100
    assert w == 3 and pairs.tolist() == [[1, 2], [5, 3]]
    w, pairs, _ = gpu.assign_1d(101, [0, 1, 100], [0, 10])  # :102-109
    assert w == 9 and pairs.tolist() == [[0, 0], [1, 10]]


def test_generalized_random_matches_reference(gpu, ref):
    rng = np.random.default_rng(0xb0b5)
    bad = []
    for it in range(600):
        np_ = int(rng.integers(1, 6))
        pos = np.sort(rng.choice(np.arange(-6, 20), np_, replace=False))
        mult = rng.integers(1, 4, np_)
        mu = np.array([rng.integers(0, m + 1) for m in mult])
        if it % 50 == 0:
            mult[0] = 0
        tg = np.sort(rng.choice(np.arange(-6, 20), int(rng.integers(0, 7)), replace=False))
        (g, eg), (r, er) = call(gpu, "assign_1d_generalized", pos, mult, mu, tg), \
            call(ref, "assign_1d_generalized", pos, mult, mu, tg)
        if eg or er:
            if eg != er:
                bad.append((it, eg, er))
            continue
        if not (g[0] == r[0] and np.array_equal(g[1], r[1]) and np.array_equal(g[2], r[2])):
            bad.append(it)
    assert not bad, bad[:3]


def test_dense_4096_chain(gpu, ref):
    # test_exact1d.cpp:575-586 shape: arbitrary (non-band) targets
    rng = np.random.default_rng(0xb16b16)
    n = 4096
    S = rng.choice(n, n * 3 // 5, replace=False)
    T = rng.choice(n, n // 2, replace=False)
    g = gpu.solve_1d(n, S, T)
    r = ref.solve_1d(n, S, T)
    assert _same_chain(g, r)


def test_c2_batch_matches_reference(gpu, ref):
    n, k, count = 1024, 563, 1024
    occ = sample_chains(0x1D000000, count, n, k)
    g = gpu.solve_1d_batch(occ, count, n, 256, 767)
    r = ref.solve_1d_batch(occ, count, n, 256, 767)
    for key in g:
        assert np.array_equal(g[key], r[key]), key


def test_chain_batch_infeasible_status(gpu):
    occ = sample_chains(7, 4, 64, 10)
    out = gpu.solve_1d_batch(occ, 4, 64, 10, 40)
    assert (out["status"] == 2).all()


def test_band_batch_sweep_stress(gpu, ref):
    """Batched band kernel vs the reference over many shapes and loadings,
    from barely feasible (long certification sweeps, many blocks, cost ties)
    to dense."""
    rng = np.random.default_rng(0xc4a1)
    for _ in range(150):
        n = int(rng.integers(8, 700))
        w = int(rng.integers(1, n + 1))
        tl = int(rng.integers(0, n - w + 1))
        k = int(rng.integers(w, n + 1)) if rng.integers(0, 2) else min(n, w + int(rng.integers(0, 4)))
        count = 256
        occ = sample_chains(int(rng.integers(0, 1 << 30)), count, n, k)
        g = gpu.solve_1d_batch(occ, count, n, tl, tl + w - 1)
        r = ref.solve_1d_batch(occ, count, n, tl, tl + w - 1)
        for key in g:
            assert np.array_equal(g[key], r[key]), (n, w, tl, k, key)
