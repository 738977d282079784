"""Shared fixtures.

Three libraries export the same C-ABI (include/recon_b200.h):
  b200    paper_2504_06182_b200/lib/librecon_b200.so   the product (CUDA)
  oracle  oracle/librecon_oracle.so                     C restatement (checker)
  ref     oracle/_ref/librecon_ref.so                   the unmodified reference, compiled (checker)
The checkers are only ever used as checkers here.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2504_06182_b200 import LIB_PATH  # noqa: E402
from paper_2504_06182_b200.abi import ReconLib  # noqa: E402

ORACLE_LIB = os.path.join(ROOT, "oracle", "librecon_oracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "librecon_ref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _load(path, name):
    if not os.path.exists(path):
        pytest.fail(f"{name} library not built: {path} (run __graft_entry__.build())")
    return ReconLib(path, name)


@pytest.fixture(scope="session")
def oracle():
    return _load(ORACLE_LIB, "oracle")


@pytest.fixture(scope="session")
def ref():
    return _load(REF_LIB, "ref")


@pytest.fixture(scope="session")
def b200_lib():
    """The product library, loaded without touching CUDA (CPU-safe)."""
    return _load(LIB_PATH, "b200")


@pytest.fixture(scope="session")
def gpu(b200_lib):
    """The product library with a live CUDA context; GPU tests fail (not skip) without one."""
    b200_lib.ctx()
    return b200_lib


@pytest.fixture
def rng():
    return np.random.default_rng(20250406)
