"""Pins the oracle's extended filter (fekf_step, fast_filter.hpp:127-224), Box–Cox
(boxcox.hpp) and CG Γ⁻¹ (covariance.hpp:118-152) against the reference's own known-answer
tests (proj/tests/test_filters.cpp:203-357) before the GPU path is checked against it.  CPU."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import (EXPERIMENT, Problem, boxcox_np, csr_dense, dense_ekf, dense_kf, low_rank_cov, rel_err)


def test_boxcox_pair_and_derivative():  # test_filters.cpp:203-226
    s = np.linspace(0.1, 4.0, 9)
    assert rel_err(O.boxcox(2.5, O.boxcox(2.5, s, "forward"), "inverse"), s) < 1e-12
    assert O.boxcox(2.5, [1.0], "forward")[0] == 0.0
    assert abs(O.boxcox(1e6, [math.e], "forward")[0] - 1.0) < 1e-5
    eps = 1e-6
    for x in (-0.5, 0.0, 0.8, 3.0):
        num = (O.boxcox(2.5, [x + eps], "inverse")[0] - O.boxcox(2.5, [x - eps], "inverse")[0]) / (2 * eps)
        assert abs(O.boxcox(2.5, [x], "derivative")[0] - num) <= 1e-7 * abs(num)
    assert O.boxcox(1.0, [0.37], "forward")[0] == 0.37 - 1.0
    assert O.boxcox(1.0, [0.37], "inverse")[0] == 0.37 + 1.0
    assert O.boxcox(1.0, [-0.2], "derivative")[0] == 1.0
    x = np.linspace(-0.9, 3.0, 17)
    for which in ("inverse", "derivative"):
        assert rel_err(O.boxcox(2.5, x, which), boxcox_np(2.5, x, which)) < 1e-15


def test_boxcox_domain_errors():  # test_filters.cpp:228-238
    with pytest.raises(O.DomainError, match="index 1"):
        O.boxcox(2.0, [0.0, -5.0, 1.0], "inverse")
    with pytest.raises(ValueError, match="alpha must be positive"):
        O.boxcox(0.0, [1.0], "inverse")


def test_cov_solve_inverts_operator():  # covariance.hpp:118-152
    p = Problem(10, 10, 2, 4, 1, 2e-4)
    cov = p.oracle_cov()
    b = np.random.default_rng(0).standard_normal(100)
    x = O.cov_solve(cov, b)
    assert rel_err(p.gamma() @ x, b) < 1e-10
    with pytest.raises(RuntimeError, match="did not converge"):
        O.cov_solve(cov, b, tol=1e-300)


def _fekf_run(p, bc, mean0, seeds, k_rank, tol, relin=1):
    f = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), mean0)
    out = []
    for y, sd in zip(p.obs, seeds):
        f.step(y, p.sigma2, bc, k_rank=k_rank, oversampling=20, trunc_tol=tol, relinearizations=relin, seed=sd)
        out.append(f.state())
    return out


def test_fekf_reduces_to_linear_filter():  # test_filters.cpp:262-287
    p = Problem(10, 10, 2, 4, 8, 2e-4)
    m = p.h.rows
    fast = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, m, 20, 17)
    U = fast.context()["U"]
    gam = p.gamma()
    ext = _fekf_run(p, 1.0, np.full(100, -1.0), [W.derive_seed(900, k) for k in range(8)], m, 0.0)
    for k, y in enumerate(p.obs):
        fast.step(y)
        fs = fast.state()
        es = ext[k]
        assert rel_err(es["mean"] + 1.0, fs["mean"]) < 1e-8
        assert rel_err(low_rank_cov(es["alpha"], es["w"], es["d"], gam),
                       low_rank_cov(fs["alpha"], U, fs["d"], gam)) < 1e-8


@pytest.mark.parametrize("relin", [1, 3])
def test_fekf_matches_dense_ekf(relin):  # test_filters.cpp:289-337
    kern = dict(EXPERIMENT, theta=1e-4)
    p = Problem(8, 8, 2, 4, 5 if relin == 1 else 3, 2e-4, kernel=kern)
    bc = 2.0 if relin == 1 else 4.0
    mean0 = np.full(64, O.boxcox(bc, [1e-4], "forward")[0])
    ext = _fekf_run(p, bc, mean0, [W.derive_seed(901 + (relin > 1), k) for k in range(len(p.obs))], p.h.rows, 0.0,
                    relin)
    dense = dense_ekf(p.gamma(), csr_dense(p.h), p.obs, p.sigma2, bc, mean0, relin)
    for es, (dm, dc) in zip(ext, dense):
        assert rel_err(es["mean"], dm) < 1e-6
        if relin == 1:
            assert rel_err(low_rank_cov(es["alpha"], es["w"], es["d"], p.gamma()), dc) < 1e-6
        assert es["d"].min() >= 0.0 and es["d"].max() < es["alpha"]


def test_fekf_truncation_bounds_rank():  # test_filters.cpp:339-357
    kern = dict(EXPERIMENT, theta=1e-5, power=1.0)
    p = Problem(12, 12, 3, 8, 6, 2e-4, kernel=kern)
    mean0 = np.full(144, O.boxcox(2.0, [1e-4], "forward")[0])
    ext = _fekf_run(p, 2.0, mean0, [W.derive_seed(903, k) for k in range(6)], p.h.rows, 1e-5)
    prev = 0
    for es in ext:
        r = len(es["d"])
        assert r <= prev + p.h.rows and r <= 144
        prev = r
    assert prev < 6 * p.h.rows


def test_fekf_errors():  # fast_filter.hpp:145-160
    p = Problem(6, 6, 2, 2, 1, 2e-4)
    f = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), np.zeros(36))
    with pytest.raises(ValueError, match="relinearizations"):
        f.step(p.obs[0], p.sigma2, 2.0, relinearizations=0)
    with pytest.raises(ValueError, match="sigma2"):
        f.step(p.obs[0], -1.0, 2.0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        f.step(p.obs[0][:2], p.sigma2, 2.0)
    g = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), np.full(36, -5.0))
    with pytest.raises(O.DomainError, match="derivative domain violation at index 0"):
        g.step(p.obs[0], p.sigma2, 2.0)
