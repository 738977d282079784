"""The B200 path reproduces the golden fixtures generated from the reference."""
import pytest

from golden_check import check_chain_fixture, check_grid_fixture, grid_fixtures

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", grid_fixtures())
def test_gpu_grid_golden(gpu, name):
    check_grid_fixture(gpu, name)


def test_gpu_chain_golden(gpu):
    check_chain_fixture(gpu)
