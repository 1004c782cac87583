"""Full-length parity on every BASELINE config (c0 10, c1 20, c2 30, c3 30, c4 50 steps):
every step's mean, d, α, diag Σ (c0/c1/c3/c4) and the 8 realizations (c3) against the CPU
oracle within 1e-9 (fast_filter.hpp:84-125, uq.hpp:16-112), the default Woodbury/PCG solver
plus the reference-order LLT solver at c1 and c2; λ normwise and per-eigenvalue."""
import pytest

from tests.parity import assert_parity, run_config, run_config_batch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_length_parity_default_solver(name):
    assert_parity(run_config(name, solver=1))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_full_length_parity_reference_llt(name):
    assert_parity(run_config(name, solver=0))


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_full_length_parity_batch(name):
    """every step of one fkb_fkf_run / fkb_fkf_run_uq call against the oracle's step-by-step
    states (the steps carry the image H·mean = y − σ²z instead of recomputing it)"""
    assert_parity(run_config_batch(name))


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_full_length_parity_pipelined_batch(name, monkeypatch):
    """the same with FKB_PIPED=1: step t's N-space mean side runs beside step t+1's m-space
    chain (the PCG cluster launched first, waiting for rotate_in's partials)"""
    monkeypatch.setenv("FKB_PIPED", "1")
    assert_parity(run_config_batch(name))
