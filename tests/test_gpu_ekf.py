"""GPU parity for the extended fast filter (fekf_step, fast_filter.hpp:127-224) against the
CPU oracle's restatement (oracle/fastkf_oracle.cpp: column MGS with CG Γ⁻¹, as the
reference) on the reference's own fekf test problems (proj/tests/test_filters.cpp:262-357),
plus the carried Γ⁻¹W and the error contract."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import EXPERIMENT, Problem, csr_dense, dense_ekf, low_rank_cov, rel_err

pytestmark = pytest.mark.gpu


def _pair(p, mean0):
    cov = P.CovarianceOperator(p.grid, p.spec())
    g = P.ExtendedFilter(cov, p.h, mean0)
    o = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), mean0)
    return cov, g, o


def _compare(p, gs, os_, tol, mean0=None):
    gam = p.gamma()
    assert gs["alpha"] == os_["alpha"] and gs["step"] == os_["step"]
    e_mean = rel_err(gs["mean"], os_["mean"])
    if mean0 is not None:  # the update itself (the means sit on a large constant offset)
        e_inc = rel_err(gs["mean"] - mean0, os_["mean"] - mean0)
        assert e_inc < tol, e_inc
    e_cov = rel_err(low_rank_cov(gs["alpha"], gs["w"], gs["d"], gam), low_rank_cov(os_["alpha"], os_["w"], os_["d"], gam))
    assert e_mean < tol, e_mean
    assert e_cov < tol, e_cov
    # the dominant modes agree one by one (d sorted descending on both sides)
    big = os_["d"] > 1e-6 * os_["alpha"]
    k = int(big.sum())
    assert np.max(np.abs(gs["d"][:k] - os_["d"][:k])) <= tol * os_["alpha"]
    return e_mean, e_cov


@pytest.mark.parametrize("case", ["identity", "boxcox2", "relin3", "trunc"])
def test_fekf_matches_oracle(case):
    if case == "identity":  # test_filters.cpp:262-287
        p, bc, tol, relin, seedtag = Problem(10, 10, 2, 4, 8, 2e-4), 1.0, 0.0, 1, 900
        mean0 = np.full(100, -1.0)
    elif case == "boxcox2":  # :289-313
        p, bc, tol, relin, seedtag = Problem(8, 8, 2, 4, 5, 2e-4, kernel=dict(EXPERIMENT, theta=1e-4)), 2.0, 0.0, 1, 901
        mean0 = np.full(64, O.boxcox(2.0, [1e-4], "forward")[0])
    elif case == "relin3":  # :315-337
        p, bc, tol, relin, seedtag = Problem(8, 8, 2, 4, 3, 2e-4), 4.0, 0.0, 3, 902
        mean0 = np.full(64, O.boxcox(4.0, [1e-4], "forward")[0])
    else:  # :339-357
        p, bc, tol, relin, seedtag = (Problem(12, 12, 3, 8, 6, 2e-4, kernel=dict(EXPERIMENT, theta=1e-5, power=1.0)),
                                      2.0, 1e-5, 1, 903)
        mean0 = np.full(144, O.boxcox(2.0, [1e-4], "forward")[0])
    cov, g, o = _pair(p, mean0)
    m = p.h.rows
    for k, y in enumerate(p.obs):
        seed = W.derive_seed(seedtag, k)
        g.step(y, p.sigma2, P.BoxCox(bc), P.FekfOptions(k_rank=m, oversampling=20, trunc_tol=tol,
                                                          relinearizations=relin, seed=seed))
        o.step(y, p.sigma2, bc, k_rank=m, oversampling=20, trunc_tol=tol, relinearizations=relin, seed=seed)
        gs, os_ = g.state(), o.state()
        _compare(p, gs, os_, 1e-9, mean0)
        # carried W̄ = Γ⁻¹W and Γ⁻¹-orthonormality of W
        if gs["w"].shape[1]:
            gam = p.gamma()
            assert rel_err(gam @ gs["wbar"], gs["w"]) < 1e-10
            assert np.max(np.abs(gs["w"].T @ gs["wbar"] - np.eye(gs["w"].shape[1]))) < 1e-10


def test_fekf_identity_equals_gpu_fkf():  # test_filters.cpp:262-287 against the GPU constant-H filter
    p = Problem(10, 10, 2, 4, 8, 2e-4)
    m = p.h.rows
    cov = P.CovarianceOperator(p.grid, p.spec())
    ctx = P.fkf_init(cov, p.h, p.sigma2, m, 20, 17)
    g = P.ExtendedFilter(cov, p.h, np.full(100, -1.0))
    gam = p.gamma()
    for k, y in enumerate(p.obs):
        st = P.fkf_step(ctx, y)
        g.step(y, p.sigma2, P.BoxCox(1.0), P.FekfOptions(k_rank=m, trunc_tol=0.0, seed=W.derive_seed(900, k)))
        es = g.state()
        assert rel_err(es["mean"] + 1.0, st["mean"]) < 1e-8
        assert es["alpha"] == st["alpha"]


def test_fekf_dense_ekf_mid_size():
    """A 24×24 grid (m = 48, three relinearizations, Box–Cox 3) against the numpy dense EKF
    (dense_filter.hpp:68-106) and the oracle."""
    p = Problem(24, 24, 6, 8, 3, 1e-4, kernel=dict(EXPERIMENT, theta=1e-4))
    mean0 = np.full(576, O.boxcox(3.0, [1e-4], "forward")[0])
    cov, g, o = _pair(p, mean0)
    dense = dense_ekf(p.gamma(), csr_dense(p.h), p.obs, p.sigma2, 3.0, mean0, 3)
    for k, (y, (dm, dc)) in enumerate(zip(p.obs, dense)):
        seed = W.derive_seed(904, k)
        g.step(y, p.sigma2, P.BoxCox(3.0), P.FekfOptions(k_rank=48, trunc_tol=0.0, relinearizations=3, seed=seed))
        o.step(y, p.sigma2, 3.0, k_rank=48, trunc_tol=0.0, relinearizations=3, seed=seed)
        gs = g.state()
        _compare(p, gs, o.state(), 1e-9, mean0)
        assert rel_err(gs["mean"], dm) < 1e-6


def test_fekf_errors_leave_state():
    p = Problem(6, 6, 2, 2, 2, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    g = P.ExtendedFilter(cov, p.h, np.zeros(36))
    g.step(p.obs[0], p.sigma2, P.BoxCox(2.0), P.FekfOptions(k_rank=4, seed=1))
    before = g.state()
    with pytest.raises(ValueError, match="relinearizations"):
        g.step(p.obs[1], p.sigma2, P.BoxCox(2.0), P.FekfOptions(relinearizations=0))
    with pytest.raises(ValueError, match="sigma2"):
        g.step(p.obs[1], 0.0, P.BoxCox(2.0))
    with pytest.raises(ValueError, match="dimension mismatch"):
        g.step(p.obs[1][:2], p.sigma2, P.BoxCox(2.0))
    with pytest.raises(ValueError, match="alpha must be positive"):
        g.step(p.obs[1], p.sigma2, P.BoxCox(0.0))
    after = g.state()
    assert after["alpha"] == before["alpha"] and np.array_equal(after["mean"], before["mean"])
    assert np.array_equal(after["d"], before["d"])
    h = P.ExtendedFilter(cov, p.h, np.full(36, -5.0))
    with pytest.raises(P.DomainError, match="derivative domain violation at index 0"):
        h.step(p.obs[0], p.sigma2, P.BoxCox(2.0))
    o = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), np.full(36, -5.0))
    with pytest.raises(O.DomainError, match="derivative domain violation at index 0"):
        o.step(p.obs[0], p.sigma2, 2.0)
    # the same step succeeds afterwards and matches the oracle
    g.step(p.obs[1], p.sigma2, P.BoxCox(2.0), P.FekfOptions(k_rank=4, seed=2))
    assert g.state()["step"] == 2


def test_fekf_c0_first_step_matches_oracle():
    """BASELINE c0 size (N = 4,096, m = 256, rank cap 256 = full rank, Box–Cox 2 about s = 1):
    the first extended step (linearization, m×m LLT, GHEP; add_low_rank returns (U, λ) from
    the zero start, so the oracle's CG Γ⁻¹ is not needed) against the oracle."""
    w, h, ys, s2 = W.problem("c0", 1)
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
    mean0 = np.zeros(w.N)  # forward(1.0) = 0 for Box–Cox 2
    k, p = w.ghep_sizes()
    g = P.ExtendedFilter(cov, h, mean0)
    g.step(ys[0], s2, P.BoxCox(2.0), P.FekfOptions(k_rank=k, oversampling=p, trunc_tol=1e-5, seed=w.ghep_seed))
    o = O.ExtendedFilter(O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu),
                         O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val), mean0)
    o.step(ys[0], s2, 2.0, k_rank=k, oversampling=p, trunc_tol=1e-5, seed=w.ghep_seed)
    gs, os_ = g.state(), o.state()
    assert gs["alpha"] == os_["alpha"] == 1.0
    assert rel_err(gs["mean"], os_["mean"]) < 1e-9
    kk = min(len(gs["d"]), len(os_["d"]))
    assert np.max(np.abs(gs["d"][:kk] - os_["d"][:kk])) <= 1e-9 * gs["alpha"]
    # W D Wᵀ applied to probe vectors (N² is too large to form)
    z = np.random.default_rng(0).standard_normal((w.N, 4))
    wg = gs["w"] @ (gs["d"][:, None] * (gs["w"].T @ z))
    wo = os_["w"] @ (os_["d"][:, None] * (os_["w"].T @ z))
    assert rel_err(wg, wo) < 1e-9


def test_fekf_trace_and_entropy():  # uq.hpp:25-53 on the extended state
    p = Problem(12, 12, 3, 8, 3, 2e-4, kernel=dict(EXPERIMENT, theta=1e-5, power=1.0))
    mean0 = np.full(144, O.boxcox(2.0, [1e-4], "forward")[0])
    cov, g, o = _pair(p, mean0)
    theta = p.kernel["theta"]
    for k, y in enumerate(p.obs):
        seed = W.derive_seed(906, k)
        g.step(y, p.sigma2, P.BoxCox(2.0), P.FekfOptions(k_rank=p.h.rows, trunc_tol=1e-5, seed=seed))
        o.step(y, p.sigma2, 2.0, k_rank=p.h.rows, trunc_tol=1e-5, seed=seed)
        so = o.state()
        tr = so["alpha"] * 144 * theta - np.sum(so["d"] * np.sum(so["w"] ** 2, axis=0))
        ent = 0.5 * ((144 - len(so["d"])) * np.log(so["alpha"]) + np.sum(np.log(so["alpha"] - so["d"])))
        assert abs(g.trace_criterion() - tr) <= 1e-9 * abs(tr)
        assert abs(g.relative_entropy() - ent) <= 1e-9 * abs(ent)
