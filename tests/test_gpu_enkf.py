"""GPU parity for the ensemble Kalman filter (enkf_step, enkf.hpp:49-94) against the CPU
oracle's restatement on the same seeds — the reference's own EnKF tests
(proj/tests/test_enkf.cpp:42-106) plus BASELINE c0-size ensembles — and its error contract."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import Problem, csr_dense, dense_kf, kernel_fn, kernel_matrix, plume_field, rel_err, \
    simulate_observations

pytestmark = pytest.mark.gpu
UNIT = dict(family=0, theta=1.0, length=0.2, power=1.0)


def _run(p, ne, ys, sigma2, seeds):
    cov = P.CovarianceOperator(p.grid, p.spec())
    ens = P.Ensemble(cov, p.h, ne)
    ocov, oh = p.oracle_cov(), p.oracle_h()
    x = np.zeros((p.nx * p.ny, ne))
    errs = []
    for y, sd in zip(ys, seeds):
        ens.step(y, sigma2, sd)
        x = O.enkf_step(x, oh, y, ocov, sigma2, sd)
        g = ens.members
        errs.append(rel_err(g, x))
        assert rel_err(ens.mean(), x.mean(axis=1)) < 1e-9
    return ens, x, max(errs)


@pytest.mark.parametrize("case", ["desk6_50", "desk10_2000", "c0_100", "c1_12", "c2_20", "c4_10"])
def test_enkf_matches_oracle(case):
    if case == "desk6_50":  # test_enkf.cpp:42-53 geometry, three cycles
        p = Problem(6, 6, 2, 3, 0, 2e-4, kernel=UNIT)
        ys = [O.gaussian_vector(p.h.rows, 5 + k) for k in range(3)]
        ne, sigma2, seeds = 50, 2e-4, [11, 12, 13]
    elif case == "desk10_2000":  # test_enkf.cpp:69-96 (N_e > m: the reference product order)
        p = Problem(10, 10, 3, 8, 0, 2e-4, kernel=dict(UNIT, theta=1e-4, power=0.5))
        ys = [simulate_observations(p.h, plume_field(10, 10, 3.0 * k), 2e-4, W.derive_seed(55, k)) for k in (1, 2, 3)]
        ne, sigma2, seeds = 2000, 2e-4, [W.derive_seed(56, k) for k in (1, 2, 3)]
    elif case in ("c2_20", "c4_10"):  # full BASELINE sizes (c2: two ray blocks; c4: 1024² torus), few members
        cfg, ne = case.split("_")
        w, h, ys_all, s2 = W.problem(cfg, 1)

        class _P:  # the workload's own operator (c2 stacks two layouts, beyond cross_well)
            nx = ny = w.n
            grid = P.Grid(w.n, w.n)
            sigma2 = s2

            def __init__(self):
                self.h = h

            def spec(self):
                return P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)

            def oracle_cov(self):
                return O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu)

            def oracle_h(self):
                return O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val)
        p = _P()
        ys, ne, sigma2, seeds = ys_all[:1], int(ne), s2, [W.derive_seed(1011, 1)]
    elif case == "c1_12":  # BASELINE c1 (512² torus: the register-resident sampler path), odd pair count
        w, h, ys_all, s2 = W.problem("c1", 1)
        p = Problem(128, 128, 32, 32, 0, s2, kernel=dict(family=1, theta=w.theta, length=w.length, nu=w.nu))
        assert np.array_equal(p.h.col, h.col)
        ys, ne, sigma2, seeds = ys_all[:1], 11, s2, [W.derive_seed(1011, 1)]
    else:  # BASELINE c0 grid and rays (N = 4096, m = 256), N_e = 100 ≤ m: the reassociated update
        w, h, ys_all, s2 = W.problem("c0", 2)
        p = Problem(64, 64, 16, 16, 0, s2, kernel=dict(family=1, theta=w.theta, length=w.length, nu=w.nu))
        assert np.array_equal(p.h.col, h.col)
        ys, ne, sigma2, seeds = ys_all[:2], 100, s2, [W.derive_seed(1011, k) for k in (1, 2)]
    ens, x, err = _run(p, ne, ys, sigma2, seeds)
    assert err < 1e-9, err


def test_enkf_statistics_and_determinism():  # test_enkf.cpp:42-53, 69-96 on the GPU path
    kern = dict(UNIT, theta=1e-4, power=0.5)
    p = Problem(10, 10, 3, 8, 0, 2e-4, kernel=kern)
    cov = P.CovarianceOperator(p.grid, p.spec())
    ys = [simulate_observations(p.h, plume_field(10, 10, 3.0 * k), 2e-4, W.derive_seed(55, k)) for k in (1, 2, 3)]
    a, b = P.Ensemble(cov, p.h, 2000), P.Ensemble(cov, p.h, 2000)
    for k, y in zip((1, 2, 3), ys):
        a.step(y, 2e-4, W.derive_seed(56, k))
        b.step(y, 2e-4, W.derive_seed(56, k))
    assert np.array_equal(a.members, b.members)
    mean, covd = dense_kf(kernel_matrix(10, 10, kernel_fn(**kern)), csr_dense(p.h), ys, 2e-4)[-1]
    se = np.sqrt(np.trace(covd) / 2000)
    assert np.linalg.norm(a.mean() - mean) <= 3.0 * se
    assert abs(np.trace(a.covariance()) - np.trace(covd)) <= 0.15 * np.trace(covd)


def test_enkf_identity_collapse():  # test_enkf.cpp:55-67
    g = P.Grid(4, 4)
    cov = P.CovarianceOperator(g, P.KernelSpec(**UNIT))
    h = P.CsrMatrix(16, 16, np.arange(17, dtype=np.int32), np.arange(16, dtype=np.int32), np.ones(16))
    y = O.gaussian_vector(16, 7)
    ens = P.Ensemble(cov, h, 200)
    ens.step(y, 0.0, 13)
    post = ens.members
    for j in range(200):
        assert np.linalg.norm(post[:, j] - y) <= 1e-8 * np.linalg.norm(y)


def test_enkf_errors():  # test_enkf.cpp:98-106, enkf.hpp:31-32,50-57,81-85
    p = Problem(4, 4, 1, 2, 0, 1e-4, kernel=UNIT)
    cov = P.CovarianceOperator(p.grid, p.spec())
    with pytest.raises(ValueError, match="at least 2"):
        P.Ensemble(cov, p.h, 1)
    ens = P.Ensemble(cov, p.h, 10)
    with pytest.raises(ValueError, match="dimension mismatch"):
        ens.step(np.zeros(5), 1e-4, 3)
    with pytest.raises(ValueError, match="nonnegative"):
        ens.step(np.zeros(2), -1.0, 3)
    # σ² = 0 with fewer members than observations: singular, members untouched
    q = Problem(8, 8, 4, 4, 0, 1e-4, kernel=UNIT)
    cq = P.CovarianceOperator(q.grid, q.spec())
    e = P.Ensemble(cq, q.h, 5)
    before = e.members
    with pytest.raises(RuntimeError, match="singular"):
        e.step(np.zeros(16), 0.0, 4)
    assert np.array_equal(e.members, before)
