"""B200-native core of the arXiv 2504.06182 atom-reconfiguration solvers.

The product is the in-tree shared library lib/librecon_b200.so (sm_100a
kernels behind the C-ABI in include/recon_b200.h).  This package holds the
build script (build_native.py), the ctypes binding of the C-ABI (abi.py),
the chunked device pipeline driver (pipeline.py), the multi-GPU sharding
(shard.py) and the input generator (inputs.py); the reference's own C++ API
is served by the C++ shim (shim/recon_shim.cpp).
"""
from __future__ import annotations

import os

from .abi import (CollisionError, InfeasibleError, InputError, LogicError, ReconError, ReconLib,
                  words_per_column)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RECON_B200_LIB") or os.path.join(PKG_DIR, "lib", "librecon_b200.so")

_native: ReconLib | None = None


def load_native() -> ReconLib:
    """Loads the CUDA library.  Fails loudly when it has not been built —
    there is no CPU fallback for the product path."""
    global _native
    if _native is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        _native = ReconLib(LIB_PATH, "b200")
    return _native


__all__ = ["load_native", "ReconLib", "ReconError", "InputError", "InfeasibleError", "CollisionError",
           "LogicError", "words_per_column", "LIB_PATH"]
