"""The C-ABI libraries load and export every entry point include/recon_b200.h
declares; without a GPU the product library fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ORACLE_LIB, REF_LIB, ROOT
from paper_2504_06182_b200 import LIB_PATH

HEADER = os.path.join(ROOT, "include", "recon_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(recon_[a-z0-9_]+)\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for n in ("recon_redrec_solve", "recon_bird_solve", "recon_solve_1d", "recon_assign_1d",
              "recon_assign_1d_generalized", "recon_batch_moves", "recon_pipeline_batch_run",
              "recon_redrec_solve_batch", "recon_solve_1d_batch", "recon_occupancy_dag"):
        assert n in names


@pytest.mark.parametrize("path", [LIB_PATH, ORACLE_LIB, REF_LIB])
def test_library_exports_every_declared_symbol(path):
    lib = C.CDLL(path)
    missing = []
    for n in declared():
        if n == "recon_sample_occ" and path != LIB_PATH:
            continue
        try:
            getattr(lib, n)
        except AttributeError:
            missing.append(n)
    assert not missing, missing


def test_product_library_is_cuda_only(b200_lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_06182_b200.abi import CudaError
    b200_lib._ctx = None
    with pytest.raises(CudaError):
        b200_lib.ctx()
    import numpy as np
    with pytest.raises(CudaError):
        b200_lib.grid_solve("redrec", np.zeros(4, np.uint64), 4, 4, 2)


def test_abi_version(b200_lib):
    assert b200_lib.lib.recon_abi_version() == 1
