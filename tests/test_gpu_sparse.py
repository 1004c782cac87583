"""GPU parity for K2 (ray-operator SpMM/SpMV): column-major and row-major block products
against a dense restatement of H on the same inputs (fast_filter.hpp:63-73, :108)."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray
from tests.helpers import Problem, csr_dense, rel_err, workload_inputs

pytestmark = pytest.mark.gpu


def _ctx(p):
    cov = P.CovarianceOperator(p.grid, p.spec())
    return P.fkf_init(cov, p.h, p.sigma2, 8, 4, 3)


@pytest.mark.parametrize("ncols", [1, 5, 33, 70, 200, 256, 300, 320, 600])
def test_spmm_layouts_match_dense(ncols):
    p = Problem(24, 20, 5, 7, 1, 2e-4)
    ctx = _ctx(p)
    Hd = csr_dense(p.h)
    m, n = Hd.shape
    rng = np.random.default_rng(ncols)
    X = rng.standard_normal((n, ncols))
    Yt = rng.standard_normal((m, ncols))
    # row-major blocks
    dX, dY = DeviceArray.from_host(np.ascontiguousarray(X).ravel()), DeviceArray(m * ncols)
    ctx.spmm_rm_device(0, dX.ptr, ncols, dY.ptr)
    assert rel_err(dY.to_host().reshape(m, ncols), Hd @ X) < 1e-13
    dYt, dZ = DeviceArray.from_host(np.ascontiguousarray(Yt).ravel()), DeviceArray(n * ncols)
    ctx.spmm_rm_device(1, dYt.ptr, ncols, dZ.ptr)
    assert rel_err(dZ.to_host().reshape(n, ncols), Hd.T @ Yt) < 1e-13
    # column-major blocks
    dXc, dYc = DeviceArray.from_host(np.asfortranarray(X).ravel(order="F")), DeviceArray(m * ncols)
    ctx.spmm_device(0, dXc.ptr, n, ncols, dYc.ptr, m)
    assert rel_err(dYc.to_host().reshape(ncols, m).T, Hd @ X) < 1e-13


def test_spmm_rm_c0_operator():
    """The BASELINE c0 ray operator (77–120 nonzeros per ray) through both layouts."""
    w, h, ys, s2 = workload_inputs("c0")
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
    ctx = P.fkf_init(cov, h, s2, 16, 4, w.ghep_seed)
    Hd = csr_dense(h)
    ncols = 276
    X = np.random.default_rng(1).standard_normal((w.N, ncols))
    dX, dY = DeviceArray.from_host(np.ascontiguousarray(X).ravel()), DeviceArray(w.m * ncols)
    ctx.spmm_rm_device(0, dX.ptr, ncols, dY.ptr)
    assert rel_err(dY.to_host().reshape(w.m, ncols), Hd @ X) < 1e-13
