"""GPU parity for the filter: GHEP (K2–K5), fkf_init/fkf_step (K6–K8) and UQ.

Desk-scale cases restate proj/tests/test_lowrank.cpp:117-144, test_filters.cpp:115-201
and test_uq.cpp:46-101; BASELINE configs compare against the CPU oracle step by step
with the north-star tolerance (≤ 1e-9 relative, FP64)."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from tests.helpers import Problem, csr_dense, dense_ghep, dense_kf, rel_err, workload_inputs

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _ghep_problem():
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    return p


def test_ghep_matches_dense_and_oracle():  # test_lowrank.cpp:117-144
    p = _ghep_problem()
    cov = P.CovarianceOperator(p.grid, p.spec())
    ctx = P.fkf_init(cov, p.h, p.sigma2, 24, 20, 19)
    assert ctx.rank() == 24
    Hd = csr_dense(p.h)
    gamma = p.gamma()
    lam_ref, _ = dense_ghep(Hd.T @ Hd / p.sigma2, gamma)
    lam = ctx.lam
    assert np.all(np.abs(lam - lam_ref[:24]) / lam_ref[:24] < 1e-8)
    assert np.all(np.diff(lam) <= 0) and lam[-1] >= 0
    U = ctx.U()
    gram = U.T @ np.linalg.solve(gamma, U)
    assert np.linalg.norm(gram - np.eye(24)) < 1e-10
    lo, Uo, _, _ = O.randomized_ghep(p.oracle_cov(), p.oracle_h(), p.sigma2, 24, 20, 19)
    assert np.max(np.abs(lam - lo)) / lo[0] < TOL
    # Ū = Γ⁻¹U
    assert rel_err(gamma @ ctx.Ubar(), U) < 1e-10


def test_offline_reconstruction_and_cross_covariance():  # test_filters.cpp:115-128
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    ctx = P.fkf_init(cov, p.h, p.sigma2, 24, 20, 5)
    Hd = csr_dense(p.h)
    A = Hd.T @ Hd / p.sigma2
    gamma = p.gamma()
    gu = np.linalg.solve(gamma, ctx.U())
    recon = gu @ np.diag(ctx.lam) @ gu.T
    assert np.linalg.norm(recon - A) <= 1e-8 * np.linalg.norm(A)
    G = Hd @ gamma @ Hd.T
    assert rel_err(ctx.h_gamma_ht(), G) < 1e-11
    assert rel_err(ctx.h_u(), Hd @ ctx.U()) < 1e-12


def test_zero_measurement_operator():  # test_filters.cpp:130-145
    g = P.Grid(6, 6)
    cov = P.CovarianceOperator(g, P.KernelSpec(family=0, theta=1e-4, length=0.2, power=0.5))
    h = P.CsrMatrix(4, 36, np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0))
    ctx = P.fkf_init(cov, h, 2e-4, 4, 10, 7)
    assert ctx.rank() == 0
    st = P.fkf_step(ctx, np.zeros(4))
    assert st["alpha"] == 1.0 and st["rank"] == 0 and np.linalg.norm(st["mean"]) == 0.0


def test_first_step_diagonal_closed_form():  # test_filters.cpp:147-160
    p = Problem(10, 10, 2, 4, 1, 2e-4)
    ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, 8, 20, 9)
    assert ctx.rank() == 8
    st = P.fkf_step(ctx, p.obs[0])
    lam = ctx.lam
    assert np.all(np.abs(st["d"] - lam / (1 + lam)) <= 1e-12 * lam / (1 + lam))


def test_full_rank_tracks_dense_kf():  # test_filters.cpp:162-191
    p = Problem(12, 12, 3, 8, 10, 2e-4)
    ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, p.h.rows, 20, 11)
    assert ctx.rank() == p.h.rows
    gamma = p.gamma()
    ref = dense_kf(gamma, csr_dense(p.h), p.obs, p.sigma2)
    U = ctx.U()
    d_prev = np.zeros(p.h.rows)
    for k, y in enumerate(p.obs):
        st = P.fkf_step(ctx, y)
        mean_ref, cov_ref = ref[k]
        assert rel_err(st["mean"], mean_ref) < 1e-8
        sigma = st["alpha"] * gamma - U @ np.diag(st["d"]) @ U.T
        assert rel_err(sigma, cov_ref) < 1e-8
        assert st["alpha"] == k + 1
        assert st["d"].min() >= 0 and st["d"].max() < st["alpha"]
        assert np.all(st["d"] >= d_prev - 1e-14)
        d_prev = st["d"]


def test_rejects_mismatched_state_rank():  # test_filters.cpp:193-201
    p = Problem(6, 6, 2, 3, 1, 2e-4)
    ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, 6, 10, 13)
    with pytest.raises(ValueError):
        ctx.set_state(1.0, np.full(2, 0.1), np.zeros(36))
    with pytest.raises(ValueError):
        ctx.step(np.zeros(p.h.rows + 1))


def test_rank_zero_uq():  # test_uq.cpp:46-58
    g = P.Grid(5, 5)
    cov = P.CovarianceOperator(g, P.KernelSpec(family=0, theta=1e-4, length=0.2, power=0.5))
    h = P.build_H(g, P.SourceReceiverLayout.cross_well(g, 2, 2))
    ctx = P.fkf_init(cov, h, 2e-4, 4, 10, 7)
    ctx.set_state(2.0, np.zeros(0), np.zeros(25))
    assert rel_err(ctx.variance(), np.full(25, 2e-4)) < 1e-14
    assert abs(ctx.trace_criterion() - 2.0 * 25 * 1e-4) <= 1e-14 * 5e-3
    ctx.set_state(1.0, np.zeros(0), np.zeros(25))
    assert ctx.relative_entropy() == 0.0


def test_offline_eigendecomposition_of_g():
    """G = HΓHᵀ = P·diag(θ)·Pᵀ with P orthogonal (block Jacobi, eig.cu)."""
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, 24, 20, 5)
    th, Pm = ctx.g_eig()
    G = ctx.h_gamma_ht()
    assert np.linalg.norm(Pm.T @ Pm - np.eye(p.h.rows)) < 1e-13
    assert np.linalg.norm(Pm @ np.diag(th) @ Pm.T - G) < 1e-14 * np.linalg.norm(G)
    assert np.allclose(np.sort(th), np.linalg.eigvalsh(G), rtol=1e-12, atol=1e-15 * np.abs(th).max())


@pytest.mark.parametrize("solver", [0, 1])
def test_solvers_agree_on_desk_problem(solver):
    p = Problem(12, 12, 3, 8, 6, 2e-4)
    ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, 16, 20, 3)
    ctx.set_solver(solver)
    of = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 16, 20, 3)
    for y in p.obs:
        st = P.fkf_step(ctx, y)
        of.step(y)
        so = of.state()
        assert rel_err(st["mean"], so["mean"]) < TOL
        assert np.max(np.abs(st["d"] - so["d"])) / so["alpha"] < TOL


def _run_both(name, steps, uq=False, realizations=0, solver=1):
    w, h, ys, s2 = workload_inputs(name, steps)
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(**kern))
    ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    ctx.set_solver(solver)
    ocov = O.CovarianceOperator(w.n, w.n, **kern)
    oh = O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val)
    of = O.FastFilter(ocov, oh, s2, k, p, w.ghep_seed)
    assert ctx.rank() == of.rank
    lo = of.context()["lam"]
    assert np.max(np.abs(ctx.lam - lo)) / lo[0] < TOL
    worst = dict(mean=0.0, d=0.0, var=0.0, real=0.0)
    for y in ys:
        st = P.fkf_step(ctx, y)
        of.step(y)
        so = of.state()
        assert st["alpha"] == so["alpha"]
        worst["mean"] = max(worst["mean"], rel_err(st["mean"], so["mean"]))
        worst["d"] = max(worst["d"], np.max(np.abs(st["d"] - so["d"])) / so["alpha"])
        if uq:
            worst["var"] = max(worst["var"], rel_err(ctx.variance(), of.variance()))
        if realizations:
            xg = ctx.realizations(w.sample_seed, realizations)
            xo = of.realizations(w.sample_seed, realizations)
            worst["real"] = max(worst["real"], max(rel_err(xg[:, j] - so["mean"], xo[:, j] - so["mean"])
                                                   for j in range(realizations)))
    return worst


@pytest.mark.parametrize("solver", [0, 1])
def test_c0_parity_all_steps(solver):
    worst = _run_both("c0", None, uq=True, realizations=2, solver=solver)
    assert worst["mean"] < TOL, worst
    assert worst["d"] < TOL, worst
    assert worst["var"] < TOL, worst
    assert worst["real"] < TOL, worst


# c1–c4 against the oracle: every step of every config, per call, as one batch and as the
# pipelined batch, in tests/test_gpu_parity_full.py (the oracle trajectory of a config is
# computed once per session there; the first-steps subsets that used to live here repeated
# c4's 80 s oracle initialization).


def test_combined_uq_call_matches_separate_calls():
    """fkb_realizations_with_variance (one U pass) ≡ fkb_variance + fkb_realizations."""
    import ctypes as C
    from paper_1405_2276_b200._native import lib
    w, h, ys, s2 = workload_inputs("c0", 3)
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
    k, p = w.ghep_sizes()
    ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    for y in ys:
        P.fkf_step(ctx, y)
    x = np.empty(w.N * 4)
    v = np.empty(w.N)
    assert lib().fkb_realizations_with_variance(ctx._f, 7, 4, C.c_void_p(x.ctypes.data), C.c_void_p(v.ctypes.data)) == 0
    assert np.array_equal(v, ctx.variance())
    assert np.array_equal(x.reshape(4, w.N).T, ctx.realizations(7, 4))


def test_step_state_round_trip_matches_step_then_state():
    """fkb_fkf_step_state (step + new state, one sync) ≡ fkb_fkf_step followed by fkb_filter_state."""
    import ctypes as C
    from paper_1405_2276_b200._native import lib
    w, h, ys, s2 = workload_inputs("c0", 4)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    a = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    for y in ys:
        sa = P.fkf_step(a, y)
        y = np.ascontiguousarray(y)
        alpha, d, mean = C.c_double(), np.empty(b.rank()), np.empty(w.N)
        assert lib().fkb_fkf_step_state(b._f, C.c_void_p(y.ctypes.data), len(y), C.byref(alpha),
                                        C.c_void_p(d.ctypes.data), C.c_void_p(mean.ctypes.data)) == 0
        assert alpha.value == sa["alpha"]
        assert np.array_equal(d, sa["d"]) and np.array_equal(mean, sa["mean"])
    bad = np.zeros(3)
    assert lib().fkb_fkf_step_state(b._f, C.c_void_p(bad.ctypes.data), 3, None, None, None) == 1  # invalid_argument


@pytest.mark.parametrize("solver", [0, 1])
def test_step_state_pinned_buffers_written_by_the_graph(solver):
    """Page-locked output buffers take the zero-copy path (the graph's last kernels write mean,
    d and the failure flag into mapped host memory): identical to the copy path, also when
    pinned, pageable and device-only steps alternate, and singularity still raises."""
    import ctypes as C
    import torch
    from paper_1405_2276_b200._native import lib
    w, h, ys, s2 = workload_inputs("c0", 6)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    a = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    a.set_solver(solver)
    b.set_solver(solver)
    pin_d = torch.empty(max(b.rank(), 1), dtype=torch.float64).pin_memory()
    pin_m = torch.empty(w.N, dtype=torch.float64).pin_memory()
    for i, y in enumerate(ys):
        sa = P.fkf_step(a, y)
        y = np.ascontiguousarray(y)
        alpha = C.c_double()
        if i % 3 == 2:  # device-side step entry point between host-buffer steps
            sb = P.fkf_step(b, y)
            assert np.array_equal(sb["mean"], sa["mean"]) and np.array_equal(sb["d"], sa["d"])
            continue
        if i % 3 == 0:
            pin_d.fill_(np.nan)
            pin_m.fill_(np.nan)
            dptr, mptr = pin_d.data_ptr(), pin_m.data_ptr()
        else:
            d_np, m_np = np.empty(b.rank()), np.empty(w.N)
            dptr, mptr = d_np.ctypes.data, m_np.ctypes.data
        assert lib().fkb_fkf_step_state(b._f, C.c_void_p(y.ctypes.data), len(y), C.byref(alpha),
                                        C.c_void_p(dptr), C.c_void_p(mptr)) == 0
        d_out = pin_d.numpy()[: b.rank()] if i % 3 == 0 else d_np
        m_out = pin_m.numpy() if i % 3 == 0 else m_np
        assert alpha.value == sa["alpha"]
        assert np.array_equal(d_out, sa["d"]) and np.array_equal(m_out, sa["mean"])
    # a singular step through the zero-copy path raises and leaves the state untouched
    st = b.state()
    b.set_state(st["alpha"], np.full(b.rank(), 50.0 * st["alpha"]), st["mean"], st["step"])
    mid = b.state()
    bad_y = np.ascontiguousarray(ys[0])
    rc = lib().fkb_fkf_step_state(b._f, C.c_void_p(bad_y.ctypes.data), len(bad_y), None,
                                  C.c_void_p(pin_d.data_ptr()), C.c_void_p(pin_m.data_ptr()))
    assert rc == 2  # runtime_error: singular
    after = b.state()
    assert after["alpha"] == mid["alpha"] and np.array_equal(after["mean"], mid["mean"])


def _c0_ctx():
    w, h, ys, s2 = workload_inputs("c0", 4)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    return w, ys, P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)


def test_cholesky_fallback_matches_pcg():
    """With the PCG capped at 0 iterations every step takes the exact cluster-Cholesky path
    (the fallback the device flag routes to); the states agree with the PCG path."""
    w, ys, a = _c0_ctx()
    _, _, b = _c0_ctx()
    b.set_pcg_maxit(0)
    for i, y in enumerate(ys):
        sa, sb = P.fkf_step(a, y), P.fkf_step(b, y)
        if i > 0:  # step 1 has d = 0, so u = 0 and the PCG exits before its cap
            assert b.cap_stats()[1] is True and a.cap_stats()[1] is False
        assert sa["alpha"] == sb["alpha"]
        assert rel_err(sb["mean"], sa["mean"]) < 1e-12
        assert np.max(np.abs(sb["d"] - sa["d"])) / sa["alpha"] < 1e-12


@pytest.mark.parametrize("solver", [0, 1])
def test_singular_innovation_raises_and_keeps_state(solver):
    """fast_filter.hpp:104-106: a non-positive-definite S raises "singular"; the device state
    is left untouched (the step's mutating epilogues are gated on the failure flag)."""
    w, ys, ctx = _c0_ctx()
    ctx.set_solver(solver)
    P.fkf_step(ctx, ys[0])
    before = ctx.state()
    # d far above α makes S = αG − B·diag(d)·Bᵀ + σ²I indefinite
    ctx.set_state(before["alpha"], np.full(ctx.rank(), 50.0 * before["alpha"]), before["mean"], before["step"])
    mid = ctx.state()
    with pytest.raises(RuntimeError, match="singular"):
        P.fkf_step(ctx, ys[1])
    after = ctx.state()
    assert after["alpha"] == mid["alpha"] and after["step"] == mid["step"]
    assert np.array_equal(after["mean"], mid["mean"]) and np.array_equal(after["d"], mid["d"])
    # recovery: restore a valid state and step again
    ctx.set_state(before["alpha"], before["d"], before["mean"], before["step"])
    st = P.fkf_step(ctx, ys[1])
    assert st["alpha"] == before["alpha"] + 1.0


@pytest.mark.parametrize("name,count,steps", [("c0", 4, 4), ("c3", 8, 2)])
def test_fused_step_uq_matches_separate_calls(name, count, steps):
    """fkb_fkf_step_uq (the step's U pass fused with diag Σ and the realizations of the new
    state) against fkf_step followed by the separate UQ calls on a twin filter, plus a
    plain step in between (graph mode switch) and the device entry point."""
    from paper_1405_2276_b200._native import DeviceArray
    w, h, ys, s2 = workload_inputs(name, steps + 1)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    a = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    for i, y in enumerate(ys[:steps]):
        st, x, var = a.step_uq(y, w.sample_seed, count)
        sb = P.fkf_step(b, y)
        assert np.array_equal(st["d"], sb["d"]) and st["alpha"] == sb["alpha"]
        # the fused pass sums U·dc per row sequentially, the plain U pass by warp reductions
        assert rel_err(st["mean"], sb["mean"]) < 1e-11
        assert rel_err(var, b.variance()) < 1e-13
        xb = b.realizations(w.sample_seed, count)
        assert rel_err(x - st["mean"][:, None], xb - sb["mean"][:, None]) < 1e-11
        if i == 0:  # a plain step on both, then back to the fused graphs
            P.fkf_step(a, ys[steps])
            P.fkf_step(b, ys[steps])
    dy = DeviceArray.from_host(np.ascontiguousarray(ys[0]))
    dx, dv = DeviceArray(w.N * count), DeviceArray(w.N)
    a.step_uq_device(dy.ptr, w.sample_seed, count, dx.ptr, dv.ptr)
    a.sync(1)
    b.step_device(dy.ptr)
    assert rel_err(dv.to_host(), b.variance()) < 1e-13
    assert rel_err(dx.to_host().reshape(count, w.N).T, b.realizations(w.sample_seed, count)) < 1e-11


def test_fused_step_uq_mapped_host_outputs():
    """fkb_fkf_step_uq with page-locked output buffers (the fused U pass writes x, diag Σ and
    the mean through mapped host memory) ≡ the same call with pageable buffers."""
    import ctypes as C
    import torch
    from paper_1405_2276_b200._native import lib
    w, h, ys, s2 = workload_inputs("c0", 3)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    a = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(P.CovarianceOperator(P.Grid(w.n, w.n), kern), h, s2, k, p, w.ghep_seed)
    cnt = 4
    px = torch.empty(cnt * w.N, dtype=torch.float64).pin_memory()
    pv = torch.empty(w.N, dtype=torch.float64).pin_memory()
    pm = torch.empty(w.N, dtype=torch.float64).pin_memory()
    pd = torch.empty(max(a.rank(), 1), dtype=torch.float64).pin_memory()
    al = C.c_double()
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    for y in ys:
        yv = np.ascontiguousarray(y)
        assert lib().fkb_fkf_step_uq(a._f, C.c_void_p(yv.ctypes.data), w.m, w.sample_seed, cnt, vp(px), vp(pv),
                                     C.byref(al), vp(pd), vp(pm)) == 0
        st, x, var = b.step_uq(y, w.sample_seed, cnt)
        assert np.array_equal(pm.numpy(), st["mean"]) and np.array_equal(pv.numpy(), var)
        assert np.array_equal(px.numpy().reshape(cnt, w.N).T, x)
        assert np.array_equal(pd.numpy()[: a.rank()], st["d"]) and al.value == st["alpha"]


def test_ghep_residual_matches_dense():  # lowrank.hpp:215-228, test_lowrank.cpp:159-167
    """Per-pair GHEP residuals on the device (Γ⁻¹U = Ū) against a dense numpy evaluation with
    a dense Γ solve; a full-range sketch leaves residuals at rounding level."""
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    cov = P.CovarianceOperator(p.grid, p.spec())
    ctx = P.fkf_init(cov, p.h, p.sigma2, 24, 20, 5)
    res = ctx.ghep_residual()
    Hd = csr_dense(p.h)
    A = Hd.T @ Hd / p.sigma2
    U = ctx.U()
    gu = np.linalg.solve(p.gamma(), U)
    want = np.linalg.norm(A @ U - gu * ctx.lam[None, :], axis=0) / (ctx.lam * np.linalg.norm(gu, axis=0))
    assert res.shape == (ctx.rank(),)
    assert np.max(np.abs(res - want)) < 1e-7
    assert res.max() < 1e-7  # the reference's sketched bound (test_lowrank.cpp:167)


def _c2_pair(monkeypatch, steps):
    """Two c2 contexts built from the same inputs: the fused step chain (default) and the
    unfused one (FKB_FUSED_CHAIN=0: separate RHS column dots, gated Cholesky, k_woodbury_st)."""
    w, h, ys, s2 = workload_inputs("c2", steps)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), kern)
    a = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    monkeypatch.setenv("FKB_FUSED_CHAIN", "0")
    b = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    monkeypatch.delenv("FKB_FUSED_CHAIN")
    return w, ys, a, b


def test_fused_chain_matches_unfused_chain(monkeypatch):
    """The fused rotate_in → PCG(+ s̃, d/α commit) chain and the five-launch chain compute the
    same step (fast_filter.hpp:100-123): same α, d to 1e-14·α, mean to 1e-12."""
    w, ys, a, b = _c2_pair(monkeypatch, 4)
    for y in ys:
        sa, sb = P.fkf_step(a, y), P.fkf_step(b, y)
        assert sa["alpha"] == sb["alpha"] and sa["step"] == sb["step"]
        assert np.max(np.abs(sa["d"] - sb["d"])) / sa["alpha"] < 1e-14
        assert rel_err(sa["mean"], sb["mean"]) < 1e-12
    assert a.cap_stats()[1] is False


def test_unverified_pcg_reruns_exactly_in_async_batches():
    """A step whose PCG does not verify (forced: cap 0) leaves the state untouched and is rerun
    on the exact Cholesky path — also inside an asynchronous batch, where the later steps of
    the batch (no-ops behind the sticky flag) are replayed after the rerun."""
    from paper_1405_2276_b200._native import DeviceArray
    w, ys, a = _c0_ctx()
    _, _, b = _c0_ctx()
    b.set_pcg_maxit(0)
    Y = DeviceArray.from_host(np.stack(ys).ravel())
    a.steps_async(Y.ptr, len(ys), w.m)
    a.sync(len(ys))
    b.steps_async(Y.ptr, len(ys), w.m)
    b.sync(len(ys))
    sa, sb = a.state(), b.state()
    assert sa["alpha"] == sb["alpha"] and sa["step"] == sb["step"] == len(ys)
    assert rel_err(sb["mean"], sa["mean"]) < 1e-12
    assert np.max(np.abs(sb["d"] - sa["d"])) / sa["alpha"] < 1e-12
    assert b.cap_stats()[1] is True


def test_unverified_pcg_rerun_writes_mapped_outputs():
    """fkb_fkf_step_state with page-locked buffers: the graph's gated epilogues skip the
    unverified step and the exact rerun writes d and the mean through the mapped pointers."""
    import ctypes as C
    import torch
    from paper_1405_2276_b200._native import lib
    w, ys, a = _c0_ctx()
    _, _, b = _c0_ctx()
    b.set_pcg_maxit(0)
    hd = torch.empty(max(b.rank(), 1), dtype=torch.float64).pin_memory()
    hm = torch.empty(w.N, dtype=torch.float64).pin_memory()
    for y in ys:
        sa = P.fkf_step(a, y)
        y = np.ascontiguousarray(y)
        hd.fill_(np.nan)
        hm.fill_(np.nan)
        alpha = C.c_double()
        assert lib().fkb_fkf_step_state(b._f, C.c_void_p(y.ctypes.data), len(y), C.byref(alpha),
                                        C.c_void_p(hd.data_ptr()), C.c_void_p(hm.data_ptr())) == 0
        assert alpha.value == sa["alpha"]
        assert rel_err(hm.numpy(), sa["mean"]) < 1e-12
        assert np.max(np.abs(hd.numpy()[: b.rank()] - sa["d"])) / sa["alpha"] < 1e-12


@pytest.mark.parametrize("name", ["c0", "c2"])
def test_run_batch_matches_step_loop(name):
    """fkb_fkf_run (the driver's step loop in one call, each step's state copied out while the
    next step runs) returns exactly the states of fkf_step called step by step."""
    w, h, ys, s2 = workload_inputs(name, 5)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), kern)
    a = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    ref = [P.fkf_step(a, y) for y in ys]
    out = b.run(np.stack(ys))
    for t, st in enumerate(ref):
        assert out["alpha"][t] == st["alpha"]
        assert np.array_equal(out["d"][t], st["d"]) and np.array_equal(out["mean"][t], st["mean"])
    sb = b.state()
    assert sb["step"] == len(ys) and sb["alpha"] == ref[-1]["alpha"]
    assert np.array_equal(sb["mean"], ref[-1]["mean"])
    # a second batch continues from the committed state
    out2 = b.run(np.stack(ys[:2]))
    st2 = P.fkf_step(a, ys[0])
    assert np.array_equal(out2["mean"][0], st2["mean"])


def test_run_uq_batch_matches_step_uq():
    """fkb_fkf_run_uq ≡ fkb_fkf_step_uq per step: new state, diag Σ and realizations (c0)."""
    w, h, ys, s2 = workload_inputs("c0", 4)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), kern)
    a = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    out = b.run(np.stack(ys), count=3, seed=77)
    for t, y in enumerate(ys):
        st, x, var = a.step_uq(y, 77, 3)
        assert np.array_equal(out["mean"][t], st["mean"]) and np.array_equal(out["d"][t], st["d"])
        assert np.array_equal(out["var"][t], var)
        assert np.array_equal(out["x"][t], x.T)


def test_run_batch_reruns_unverified_and_raises_singular():
    """Forced PCG give-up inside a host batch: every step is rerun exactly and the outputs match
    the step loop; a singular step raises naming it and commits the steps before it."""
    w, ys, a = _c0_ctx()
    _, _, b = _c0_ctx()
    b.set_pcg_maxit(0)
    ref = [P.fkf_step(a, y) for y in ys]
    out = b.run(np.stack(ys))
    for t, st in enumerate(ref):
        assert out["alpha"][t] == st["alpha"]
        assert rel_err(out["mean"][t], st["mean"]) < 1e-12
    st = b.state()
    b.set_state(st["alpha"], np.full(b.rank(), 50.0 * st["alpha"]), st["mean"], st["step"])
    with pytest.raises(RuntimeError, match=r"singular \(step 1 of"):
        b.run(np.stack(ys[:2]))
    assert b.state()["alpha"] == st["alpha"]


def _run_pinned(ctx, ys):
    """fkb_fkf_run with page-locked input/output arrays (as bench.py's e2e leg calls it)."""
    import ctypes as C
    import torch
    from paper_1405_2276_b200._native import lib
    Y = torch.from_numpy(np.ascontiguousarray(np.stack(ys))).pin_memory()
    ns, r = Y.shape[0], max(ctx.rank(), 1)
    al = torch.full((ns,), np.nan, dtype=torch.float64).pin_memory()
    d = torch.full((ns, r), np.nan, dtype=torch.float64).pin_memory()
    mean = torch.full((ns, ctx.n), np.nan, dtype=torch.float64).pin_memory()
    rc = lib().fkb_fkf_run(ctx._f, C.c_void_p(Y.data_ptr()), ns, Y.shape[1], C.c_void_p(al.data_ptr()),
                           C.c_void_p(d.data_ptr()), r, C.c_void_p(mean.data_ptr()), ctx.n)
    return rc, dict(alpha=al.numpy().copy(), d=d.numpy()[:, : ctx.rank()].copy(), mean=mean.numpy().copy())


@pytest.mark.parametrize("name,nsteps", [("c0", 7), ("c2", 6)])
def test_run_batch_page_locked_outputs_match_step_loop(name, nsteps):
    """fkb_fkf_run with page-locked arrays — exactly the states of the step loop, for odd and
    even batch lengths and a second batch (parity flip).  (Writing the rows straight through
    mapped memory from the step's kernels measured slower than the copy stream: c2 e2e 10,835
    against 12,321 steps/s, the PCIe writes stall the last FFT pass.)"""
    w, h, ys, s2 = workload_inputs(name, nsteps)
    kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), kern)
    a = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    b = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    ref = [P.fkf_step(a, y) for y in ys]
    rc, out = _run_pinned(b, ys[: nsteps - 2])
    assert rc == 0
    rc, out2 = _run_pinned(b, ys[nsteps - 2:])
    assert rc == 0
    for t, st in enumerate(ref):
        o, i = (out, t) if t < nsteps - 2 else (out2, t - (nsteps - 2))
        assert o["alpha"][i] == st["alpha"]
        assert np.array_equal(o["d"][i], st["d"]) and np.array_equal(o["mean"][i], st["mean"])
    sb = b.state()
    assert sb["step"] == nsteps and np.array_equal(sb["mean"], ref[-1]["mean"])
    # the per-call API afterwards continues from the batch's state
    nxt_a, nxt_b = P.fkf_step(a, ys[0]), P.fkf_step(b, ys[0])
    assert np.array_equal(nxt_a["mean"], nxt_b["mean"])
    assert np.array_equal(out2["mean"][-1], ref[-1]["mean"])


def test_run_batch_page_locked_reruns_unverified_and_raises_singular():
    """Page-locked arrays with a forced PCG give-up: every step is rerun exactly and lands in its
    row; a singular step raises naming it and the state stays."""
    w, ys, a = _c0_ctx()
    _, _, b = _c0_ctx()
    b.set_pcg_maxit(0)
    ref = [P.fkf_step(a, y) for y in ys]
    rc, out = _run_pinned(b, ys)
    assert rc == 0
    for t, st in enumerate(ref):
        assert out["alpha"][t] == st["alpha"]
        assert rel_err(out["mean"][t], st["mean"]) < 1e-12
        assert np.max(np.abs(out["d"][t] - st["d"])) / st["alpha"] < 1e-12
    st = b.state()
    b.set_state(st["alpha"], np.full(b.rank(), 50.0 * st["alpha"]), st["mean"], st["step"])
    rc, _ = _run_pinned(b, ys[:2])
    from paper_1405_2276_b200._native import lib
    assert rc != 0 and "singular (step 1 of" in lib().fkb_last_error().decode()
    assert b.state()["alpha"] == st["alpha"]


def test_uncertified_capacitance_takes_the_exact_path(monkeypatch):
    """A capacitance K without the Gershgorin SPD certificate (forced: FKB_CAP_CERT=fail) is
    never trusted to the PCG: every step reruns on the exact Cholesky path, same states."""
    w, ys, a = _c0_ctx()
    monkeypatch.setenv("FKB_CAP_CERT", "fail")
    _, _, b = _c0_ctx()
    monkeypatch.delenv("FKB_CAP_CERT")
    for y in ys:
        sa, sb = P.fkf_step(a, y), P.fkf_step(b, y)
        assert sa["alpha"] == sb["alpha"]
        assert rel_err(sb["mean"], sa["mean"]) < 1e-12
        assert np.max(np.abs(sb["d"] - sa["d"])) / sa["alpha"] < 1e-12
        assert b.cap_stats()[1] is True and a.cap_stats()[1] is False
