"""The reference's OWN doctest suites (proj/tests/test_*.cpp, unmodified),
compiled against the drop-in shim (paper_2504_06182_b200/shim/recon_shim.cpp)
so every red_rec / bird / solve_1d / assign_1d* / batch_moves / occupancy_dag
call they make runs on the B200 kernels.  Binaries are built in the build
container (shim/Makefile, needs the reference sources) and travel with the repo."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "paper_2504_06182_b200", "shim", "bin")
MODULES = ["core", "oracle", "exact1d", "redrec", "bird", "batching", "aro"]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mod", MODULES)
def test_reference_suite_passes_on_b200(gpu, mod):
    exe = os.path.join(BIN, f"test_{mod}")
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (run __graft_entry__.build() where /root/reference exists)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    summary = [l for l in r.stdout.splitlines() if l.startswith("[doctest]")]
    assert r.returncode == 0, (summary, r.stderr[-3000:])
    assert summary and "| 0 failed" in summary[0], summary
