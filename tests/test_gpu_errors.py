"""The device path's error contract against the reference's: exception types
and message substrings for the validations the reference tests exercise on this path
(kernel.hpp:27-43, lowrank.hpp:145-151, fast_filter.hpp:54-57,88-95, uq.hpp:39-53)."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from tests.helpers import Problem

pytestmark = pytest.mark.gpu


def test_kernel_parameter_validation():  # test_kernel_covariance.cpp "kernel parameter validation"
    g = P.Grid(8, 8)
    with pytest.raises(ValueError, match="theta"):
        P.CovarianceOperator(g, P.KernelSpec(family=1, theta=0.0, length=0.2, nu=0.5))
    with pytest.raises(ValueError, match="length"):
        P.CovarianceOperator(g, P.KernelSpec(family=1, theta=1.0, length=-1.0, nu=0.5))
    with pytest.raises(ValueError, match="nu"):
        P.CovarianceOperator(g, P.KernelSpec(family=1, theta=1.0, length=0.2, nu=0.0))
    with pytest.raises(ValueError, match="power"):
        P.CovarianceOperator(g, P.KernelSpec(family=0, theta=1.0, length=0.2, power=2.5))


def test_ghep_size_validation():  # test_lowrank.cpp "oversized sketches are rejected"
    p = Problem(5, 5, 2, 2, 1, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    with pytest.raises(ValueError, match="exceeds problem size"):
        P.fkf_init(cov, p.h, p.sigma2, 20, 10, 1)
    with pytest.raises(ValueError, match="nonnegative"):
        P.fkf_init(cov, p.h, p.sigma2, -1, 10, 1)


def test_fkf_init_validation():  # fast_filter.hpp:54-57
    p = Problem(6, 6, 2, 3, 1, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    with pytest.raises(ValueError, match="sigma2"):
        P.fkf_init(cov, p.h, 0.0, 4, 2, 1)
    wrong = P.CsrMatrix(p.h.rows, p.h.cols + 1, p.h.rowptr, p.h.col, p.h.val)
    with pytest.raises(ValueError, match="columns"):
        P.fkf_init(cov, wrong, p.sigma2, 4, 2, 1)


def test_step_and_uq_validation():  # fast_filter.hpp:88-95, uq.hpp:39-53
    p = Problem(6, 6, 2, 3, 1, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    ctx = P.fkf_init(cov, p.h, p.sigma2, 4, 2, 1)
    with pytest.raises(ValueError, match="observation length"):
        P.fkf_step(ctx, np.zeros(p.h.rows + 1))
    with pytest.raises(ValueError, match="alpha > 0"):  # zero start: α = 0
        P.relative_entropy(ctx)
    with pytest.raises(ValueError, match="count"):
        ctx.realizations(1, 9)
    with pytest.raises(ValueError, match="rank"):
        ctx.set_state(1.0, np.zeros(ctx.rank() + 1), np.zeros(36))
    P.fkf_step(ctx, p.obs[0])
    assert np.isfinite(P.relative_entropy(ctx))


def test_cov_apply_length_validation():  # covariance.hpp apply(): expected length N
    cov = P.CovarianceOperator(P.Grid(9, 11), P.KernelSpec(family=1, theta=1.0, length=0.2, nu=1.5))
    with pytest.raises(ValueError, match="length"):
        cov.apply(np.zeros(5))
