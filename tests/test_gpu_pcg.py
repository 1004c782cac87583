"""GPU tests of the capacitance solver kernel (cappcg.cu) through its C-ABI test hook: the
pipelined Jacobi-PCG in one 16-CTA cluster against a dense solve, over every code path
(register-resident K rows for n ≤ 320 and n ≤ 512, shared-memory rows above, one or two owner
warps per CTA, CTAs without rows), and its definiteness certification (the flag that routes a
step to the exact Cholesky, which then reports "singular" like fast_filter.hpp:104-106)."""
import ctypes as C

import numpy as np
import pytest

from paper_1405_2276_b200._native import lib

pytestmark = pytest.mark.gpu


def _solve(K, b):
    n = len(b)
    x, it = np.empty(n), C.c_int()
    rc = lib().fkb_cap_pcg_test(n, np.ascontiguousarray(K.T).ravel(), np.ascontiguousarray(b), x, C.byref(it),
                                np.zeros(64, dtype=np.uint64))
    return rc, x, it.value


def _near_identity(n, seed, spread=0.05):
    # the Woodbury capacitance shape: I minus a small PSD term, plus diagonal jitter
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((n, n)) / np.sqrt(n)
    return np.eye(n) - spread * (F.T @ F) / 2 + np.diag(rng.uniform(0, 0.1, n))


@pytest.mark.parametrize("n", [1, 5, 15, 16, 17, 100, 256, 300, 319, 320, 321, 400, 480, 500, 512, 513, 700, 1024])
def test_pcg_matches_dense_solve(n):
    K = _near_identity(n, n)
    b = np.random.default_rng(n + 1).standard_normal(n)
    rc, x, it = _solve(K, b)
    assert rc == 0 and 0 < it < 200
    ref = np.linalg.solve(K, b)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-12


def _conditioned(n, kappa, seed=7):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (Q * np.geomspace(1.0 / kappa, 1.0, n)) @ Q.T, rng.standard_normal(n)


@pytest.mark.parametrize("n", [300, 500])
def test_pcg_moderately_conditioned(n):
    """κ = 10 with a spread spectrum: tens of iterations, same accuracy bar."""
    K, b = _conditioned(n, 10.0)
    rc, x, it = _solve(K, b)
    assert rc == 0 and it > 20
    ref = np.linalg.solve(K, b)
    assert np.linalg.norm(K @ x - b) / np.linalg.norm(b) < 1e-12
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("kappa", [100.0, 1e4])
def test_pcg_ill_conditioned_raises_fallback(kappa):
    """A spread spectrum with κ ≥ 100 cannot reach ‖r‖ ≤ 1e-14‖u‖ in the pipelined recurrence
    (stagnation, then η ≤ 0, or the 200-iteration cap): the kernel leaves u and raises the
    fallback flag; the step then solves with the exact cluster Cholesky."""
    K, b = _conditioned(300, kappa)
    rc, x, it = _solve(K, b)
    assert rc == 2 and 0 < it <= 200
    assert np.array_equal(x, b)  # u untouched


def test_pcg_zero_rhs_returns_zero():
    K = _near_identity(300, 3)
    rc, x, it = _solve(K, np.zeros(300))
    assert rc == 0 and np.all(x == 0.0)


@pytest.mark.parametrize("n", [16, 300, 500, 700])
def test_pcg_flags_non_positive_pivot(n):
    K = _near_identity(n, 5)
    K[n // 2, n // 2] = -1.0
    rc, _, _ = _solve(K, np.ones(n))
    assert rc == 2  # fallback raised: the exact Cholesky decides (and reports singular)


@pytest.mark.parametrize("n", [300, 500])
def test_pcg_flags_indefinite_with_positive_diagonal(n):
    """Positive diagonal but an indefinite matrix: caught by the curvature test pᵀKp ≤ 0."""
    rng = np.random.default_rng(11)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.ones(n)
    ev[:n // 3] = -0.5
    K = (Q * ev) @ Q.T
    K += np.diag(np.abs(np.diag(K)) + 0.01 - np.diag(K)) * (np.diag(K) <= 0)  # force K_ii > 0
    assert np.all(np.diag(K) > 0)
    rc, _, _ = _solve(K, rng.standard_normal(n))
    assert rc == 2


def test_pcg_repeatable_bitwise():
    K = _near_identity(300, 9)
    b = np.random.default_rng(10).standard_normal(300)
    outs = [_solve(K, b)[1] for _ in range(3)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
