"""Synthetic inputs and occ-bit packing (host helpers for tests and bench).

Seeded instances follow the reference's generator exactly:
Rng(seed).sample_without_replacement(W*H, k) (rng.hpp:49-59), implemented in
C (csrc/sample.cpp, exported as recon_sample_occ) because a 512x512 partial
Fisher-Yates per instance is too slow in Python.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import LIB_PATH


def words_per_column(h: int) -> int:
    return (h + 63) // 64


def pack_grid(occ2d: np.ndarray) -> np.ndarray:
    """occ2d[x, y] (bool, W x H) -> column-major occ bits."""
    W, H = occ2d.shape
    wpc = words_per_column(H)
    padded = np.zeros((W, wpc * 64), dtype=np.uint8)
    padded[:, :H] = occ2d
    bits = np.packbits(padded.reshape(W, wpc, 64), axis=2, bitorder="little")  # (W, wpc, 8)
    return bits.reshape(W, wpc, 8).view(np.uint64).reshape(W * wpc).copy()


def unpack_grid(occ: np.ndarray, W: int, H: int) -> np.ndarray:
    wpc = words_per_column(H)
    b = np.unpackbits(np.ascontiguousarray(occ, np.uint64).view(np.uint8).reshape(W, wpc * 8),
                      axis=1, bitorder="little")
    return b[:, :H].astype(bool)


def pack_chain(S, n: int) -> np.ndarray:
    words = (n + 63) // 64
    bits = np.zeros(words * 64, np.uint8)
    bits[np.asarray(S, np.int64)] = 1
    return np.packbits(bits, bitorder="little").view(np.uint64).copy()


def grid_from_vertices(S, W: int, H: int) -> np.ndarray:
    occ2d = np.zeros((W, H), bool)
    S = np.asarray(S, np.int64)
    occ2d[S // H, S % H] = True
    return pack_grid(occ2d)


def grid_from_depths(depths_per_column, H: int) -> np.ndarray:
    """Reference test helper band_problem (test_redrec.cpp:15-23): depth = row from the top."""
    W = len(depths_per_column)
    occ2d = np.zeros((W, H), bool)
    for x, ds in enumerate(depths_per_column):
        for d in ds:
            occ2d[x, H - 1 - d] = True
    return pack_grid(occ2d)


_lib = None


def _sampler():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.recon_sample_occ.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                          C.c_void_p, C.c_int32]
        _lib.recon_sample_occ.restype = C.c_int
    return _lib


def sample_grids(seed_base: int, count: int, W: int, H: int, k: int, threads: int = 0) -> np.ndarray:
    """count instances, instance i = Rng(seed_base + i).sample_without_replacement(W*H, k)."""
    wpc = words_per_column(H)
    out = np.zeros(count * W * wpc, np.uint64)
    st = _sampler().recon_sample_occ(seed_base, count, W, H, k, 0, out.ctypes.data, threads)
    if st != 0:
        raise RuntimeError(f"recon_sample_occ failed: {st}")
    return out


def sample_chains(seed_base: int, count: int, n: int, k: int, threads: int = 0) -> np.ndarray:
    words = (n + 63) // 64
    out = np.zeros(count * words, np.uint64)
    st = _sampler().recon_sample_occ(seed_base, count, n, 1, k, 1, out.ctypes.data, threads)
    if st != 0:
        raise RuntimeError(f"recon_sample_occ failed: {st}")
    return out
