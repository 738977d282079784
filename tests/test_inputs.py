"""The synthetic-input generator is bit-identical to the reference's Rng
(rng.hpp:14-59), and the occ-bit packing round-trips."""
import ctypes as C

import numpy as np
import pytest

from conftest import REF_LIB
from paper_2504_06182_b200.inputs import (grid_from_vertices, pack_grid, sample_chains, sample_grids,
                                          unpack_grid)


@pytest.mark.parametrize("seed,W,H,k", [(1, 32, 32, 614), (0x64000000, 64, 64, 2662), (257, 256, 256, 39322),
                                        (5, 13, 7, 50), (0x51200000, 512, 512, 157286)])
def test_sampler_matches_reference_rng(seed, W, H, k):
    ref = C.CDLL(REF_LIB)
    out = np.zeros(k, np.int32)
    ref.recon_ref_sample(C.c_uint64(seed), W * H, k, out.ctypes.data_as(C.c_void_p))
    assert np.array_equal(sample_grids(seed, 1, W, H, k), grid_from_vertices(out, W, H))


def test_chain_sampler_matches_reference_rng():
    ref = C.CDLL(REF_LIB)
    out = np.zeros(563, np.int32)
    ref.recon_ref_sample(C.c_uint64(0x1D000001), 1024, 563, out.ctypes.data_as(C.c_void_p))
    bits = np.unpackbits(sample_chains(0x1D000001, 1, 1024, 563).view(np.uint8), bitorder="little")
    assert np.array_equal(np.nonzero(bits)[0], out)


def test_pack_roundtrip():
    rng = np.random.default_rng(3)
    for W, H in [(3, 5), (7, 64), (5, 65), (4, 130)]:
        o = rng.random((W, H)) < 0.5
        assert (unpack_grid(pack_grid(o), W, H) == o).all()


def test_batched_sampler_is_seed_indexed():
    a = sample_grids(100, 3, 16, 16, 100)
    b = sample_grids(102, 1, 16, 16, 100)
    assert np.array_equal(a[2 * 16:], b)
