"""Pins the oracle's EnKF (enkf_step, enkf.hpp:43-94) against the reference's own tests
(proj/tests/test_enkf.cpp:27-106) before the GPU path is checked against it.  CPU."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import EXPERIMENT, Problem, csr_dense, dense_kf, kernel_fn, kernel_matrix, plume_field, \
    simulate_observations

UNIT = dict(family=0, theta=1.0, length=0.2, power=1.0)  # test_enkf.cpp:17-24


def _cross(n, ns, nr):
    return O.build_H(n, n, [(0.0, (i + 0.5) / ns) for i in range(ns)], [(1.0, (j + 0.5) / nr) for j in range(nr)])


def test_enkf_deterministic_per_seed():  # test_enkf.cpp:42-53
    cov = O.CovarianceOperator(6, 6, **UNIT)
    h = _cross(6, 2, 3)
    y = O.gaussian_vector(h.rows, 5)
    a = O.enkf_step(np.zeros((36, 50)), h, y, cov, 2e-4, 11)
    b = O.enkf_step(np.zeros((36, 50)), h, y, cov, 2e-4, 11)
    c = O.enkf_step(np.zeros((36, 50)), h, y, cov, 2e-4, 12)
    assert np.array_equal(a, b) and np.linalg.norm(a - c) > 0.0


def test_enkf_identity_observations_collapse():  # test_enkf.cpp:55-67
    cov = O.CovarianceOperator(4, 4, **UNIT)
    h = O.Csr.from_arrays(16, 16, np.arange(17, dtype=np.int32), np.arange(16, dtype=np.int32), np.ones(16))
    y = O.gaussian_vector(16, 7)
    post = O.enkf_step(np.zeros((16, 200)), h, y, cov, 0.0, 13)
    for j in range(200):
        assert np.linalg.norm(post[:, j] - y) <= 1e-8 * np.linalg.norm(y)


def test_enkf_large_ensemble_approaches_dense_kf():  # test_enkf.cpp:69-96
    kern = dict(UNIT, theta=1e-4, power=0.5)
    cov = O.CovarianceOperator(10, 10, **kern)
    p = Problem(10, 10, 3, 8, 0, 2e-4, kernel=kern)
    h = p.oracle_h()
    ys = [simulate_observations(p.h, plume_field(10, 10, 3.0 * k), 2e-4, W.derive_seed(55, k)) for k in (1, 2, 3)]
    x = np.zeros((100, 2000))
    for k, y in zip((1, 2, 3), ys):
        x = O.enkf_step(x, h, y, cov, 2e-4, W.derive_seed(56, k))
    mean, covd = dense_kf(kernel_matrix(10, 10, kernel_fn(**kern)), csr_dense(p.h), ys, 2e-4)[-1]
    se = np.sqrt(np.trace(covd) / 2000)
    assert np.linalg.norm(x.mean(axis=1) - mean) <= 3.0 * se
    assert abs(np.trace(np.cov(x)) - np.trace(covd)) <= 0.15 * np.trace(covd)


def test_enkf_errors():  # test_enkf.cpp:98-106, enkf.hpp:50-57
    cov = O.CovarianceOperator(4, 4, **UNIT)
    h = _cross(4, 1, 2)
    with pytest.raises(ValueError, match="dimension mismatch"):
        O.enkf_step(np.zeros((9, 10)), h, np.zeros(2), cov, 1e-4, 3)
    with pytest.raises(ValueError, match="dimension mismatch"):
        O.enkf_step(np.zeros((16, 10)), h, np.zeros(5), cov, 1e-4, 3)
    with pytest.raises(ValueError, match="at least 2"):
        O.enkf_step(np.zeros((16, 1)), h, np.zeros(2), cov, 1e-4, 3)
    with pytest.raises(ValueError, match="nonnegative"):
        O.enkf_step(np.zeros((16, 4)), h, np.zeros(2), cov, -1.0, 3)
