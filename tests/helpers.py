"""Instance generators and comparison helpers shared by the tests."""
import numpy as np

from paper_2504_06182_b200.abi import ReconError
from paper_2504_06182_b200.inputs import pack_grid


def random_band_instance(rng, max_w, max_h, critical=False):
    """Like random_band_problem (test_redrec.cpp:37-47) but with numpy draws."""
    W = int(rng.integers(1, max_w + 1))
    H = int(rng.integers(2, max_h + 1))
    hp = int(rng.integers(1, H))
    nt = W * hp
    ns = min(W * H, nt + int(rng.integers(0, W + 1))) if critical else int(rng.integers(nt, W * H + 1))
    ids = rng.choice(W * H, ns, replace=False)
    occ2d = np.zeros((W, H), bool)
    occ2d.flat[ids] = True
    return pack_grid(occ2d), W, H, hp


def call(lib, fn, *args, **kw):
    try:
        return getattr(lib, fn)(*args, **kw), None
    except ReconError as e:
        return None, (type(e).__name__, str(e))


def same_grid(a, b):
    return (np.array_equal(a.path_src, b.path_src) and np.array_equal(a.path_dst, b.path_dst)
            and np.array_equal(a.path_event, b.path_event) and a.total_displacement == b.total_displacement
            and a.displaced_tokens == b.displaced_tokens and np.array_equal(a.events, b.events)
            and ((a.dag is None and b.dag is None) or np.array_equal(a.dag, b.dag)))
