"""The C oracle reproduces the golden fixtures generated from the reference."""
import pytest

from golden_check import check_chain_fixture, check_grid_fixture, grid_fixtures


@pytest.mark.parametrize("name", grid_fixtures())
def test_oracle_grid_golden(oracle, name):
    check_grid_fixture(oracle, name)


def test_oracle_chain_golden(oracle):
    check_chain_fixture(oracle)
