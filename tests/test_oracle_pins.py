"""Pins the CPU oracle (oracle/fastkf_oracle.cpp) before it is trusted as the checker.

Every known-answer test the reference suites hold for the hot path is
restated here against the oracle, plus the independent numpy/scipy golden vectors in
tests/golden/golden.npz (make_golden.py).  CPU only."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import EXPERIMENT, Problem, csr_dense, dense_ghep, dense_kf, kernel_fn, kernel_matrix, rel_err

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
PE, MA = O.POWERED_EXPONENTIAL, O.MATERN


# ---------------------------------------------------------------- kernel.hpp (test_kernel_covariance.cpp:39-87)
def test_kernel_sill_and_closed_forms():
    assert O.kernel_eval(PE, 1e-4, 1.0, 0.0, power=0.5) == 1e-4
    assert abs(O.kernel_eval(MA, 3.5, 0.7, 0.0, nu=1.5) - 3.5) <= 1e-14 * 3.5
    assert abs(O.kernel_eval(PE, 1.0, 2.0, 2.0, power=1.0) - math.exp(-1.0)) <= 1e-14
    for r in (0.1, 0.5, 1.7, 3.0):
        assert abs(O.kernel_eval(PE, 2.5, 0.4, r, power=0.5) - 2.5 * math.exp(-math.sqrt(r / 0.4))) <= 1e-13 * 2.5
    for r in (0.01, 0.1, 0.5, 1.0, 2.0):  # Matérn ν=½ with alpha_scale ≡ exponential
        assert rel_err(O.kernel_eval(MA, 1e-4, 0.3, r, nu=0.5, alpha_scale=2.0), 1e-4 * math.exp(-2 * r)) < 1e-12
    for r in (0.05, 0.3, 1.1):
        assert rel_err(O.kernel_eval(MA, 1.0, 0.25, r, nu=0.5), math.exp(-r / 0.25)) < 1e-12


def test_kernel_golden_scipy():
    r = GOLD["kernel_r"]
    for nu in (0.5, 1.5, 2.5):
        got = np.array([O.kernel_eval(MA, 1.0, 0.15, x, nu=nu) for x in r])
        assert np.max(np.abs(got - GOLD[f"matern_nu{nu}"])) < 1e-13
    got = np.array([O.kernel_eval(PE, 2.5, 0.4, x, power=0.5) for x in r])
    assert np.max(np.abs(got - GOLD["powexp"])) < 1e-13


def test_kernel_monotone_and_validation():
    for fam, kw in [(PE, dict(power=0.5)), (PE, dict(power=2.0)), (MA, dict(nu=0.5)), (MA, dict(nu=2.5))]:
        prev = O.kernel_eval(fam, 1.0, 0.3, 0.0, **kw)
        for i in range(1, 101):
            v = O.kernel_eval(fam, 1.0, 0.3, 0.05 * i, **kw)
            assert 0.0 <= v <= prev + 1e-15
            prev = v
    for args in [(PE, -1.0, 0.2, 0.1, 0.5), (PE, 1.0, 0.0, 0.1, 0.5), (PE, 1.0, 0.2, 0.1, 2.5)]:
        with pytest.raises(ValueError):
            O.kernel_eval(args[0], args[1], args[2], args[3], power=args[4])
    with pytest.raises(ValueError):
        O.kernel_eval(MA, 1.0, 0.2, 0.1, nu=-0.5)


# ---------------------------------------------------------------- covariance.hpp FFT mode
def test_one_cell_operator():  # test_kernel_covariance.cpp:89-98
    cov = O.CovarianceOperator(1, 1, family=PE, theta=3e-3, length=0.2, power=0.5)
    assert abs(cov.apply(np.array([2.0]))[0] - 6e-3) <= 1e-13 * 6e-3


@pytest.mark.parametrize("nx,ny,lx", [(20, 20, 1.0), (13, 7, 2.0), (64, 64, 1.0)])
def test_fft_matches_dense(nx, ny, lx):  # test_kernel_covariance.cpp:100-109
    cov = O.CovarianceOperator(nx, ny, lx, 1.0, **EXPERIMENT)
    K = kernel_matrix(nx, ny, kernel_fn(**EXPERIMENT), lx, 1.0)
    for t in range(3):
        x = O.gaussian_vector(nx * ny, 11, t)
        assert rel_err(cov.apply(x), K @ x) < 1e-12


def test_fft_golden():
    for nx, ny, lx in [(20, 20, 1.0), (13, 7, 2.0)]:
        cov = O.CovarianceOperator(nx, ny, lx, 1.0, **EXPERIMENT)
        assert rel_err(cov.apply(GOLD[f"gx_{nx}x{ny}_x"]), GOLD[f"gx_{nx}x{ny}_y"]) < 1e-12


def test_columns_symmetry_trace_spectrum():  # :111-154
    cov = O.CovarianceOperator(9, 11, **EXPERIMENT)
    K = kernel_matrix(9, 11, kernel_fn(**EXPERIMENT))
    for i in (0, 40, 98):
        e = np.zeros(99)
        e[i] = 1.0
        assert rel_err(cov.apply(e), K[:, i]) < 1e-12
    big = O.CovarianceOperator(59, 55, **EXPERIMENT)
    assert abs(59 * 55 * 1e-4 - 3245e-4) < 1e-15  # trace = N·θ (covariance.hpp:180)
    assert np.all(np.isfinite(big.apply(O.gaussian_vector(59 * 55, 5))))
    c20 = O.CovarianceOperator(20, 20, **EXPERIMENT)
    sp = c20.spectrum()
    assert sp.size >= 39 * 39 and sp.min() >= 0.0
    assert (c20.mx, c20.my) == (40, 40)  # next_smooth(39) = 40


def test_embedding_failure_message():  # :304-320
    with pytest.raises(RuntimeError, match="powered-exponential.*theta"):
        O.CovarianceOperator(16, 16, family=PE, theta=1.0, length=2.0, power=2.0)


def test_next_smooth_and_baseline_tori():
    assert [O.next_smooth(n) for n in (1, 39, 117, 109, 127, 255)] == [1, 40, 120, 112, 128, 256]
    # c1 needs the doubled padding (512²), c0 128², c2/c3 512²
    for name, want in [("c0", 128), ("c1", 512)]:
        w = W.CONFIGS[name]
        cov = O.CovarianceOperator(w.n, w.n, family=MA, theta=w.theta, length=w.length, nu=w.nu)
        assert cov.mx == cov.my == want


# ---------------------------------------------------------------- rng.hpp
def test_rng_streams():
    assert O.splitmix64(0) == W.splitmix64(0)
    assert O.derive_seed(12, 3000) == W.derive_seed(12, 3000)
    for seed, stream in [(0, 0), (77, 5), (2 ** 63 + 5, 123)]:
        a = O.gaussian_vector(1001, seed, stream)
        b = W.rng_normals(1001, seed, stream)
        assert np.max(np.abs(a - b)) < 1e-13
    g = O.gaussian_matrix(50, 4, 9, 2)
    for j in range(4):
        assert np.array_equal(g[:, j], O.gaussian_vector(50, 9, 2 + j))


# ---------------------------------------------------------------- tomography.hpp (test_tomography.cpp)
def test_ray_kats():
    cells, lens = O.trace_ray(10, 5, (0.0, 0.5), (1.0, 0.5))  # horizontal through row centers
    assert len(cells) == 10 and np.allclose(lens, 0.1, rtol=1e-12)
    assert list(cells) == [i * 5 + 2 for i in range(10)]
    cells, lens = O.trace_ray(1, 1, (0.0, 0.0), (0.3, 0.4), lx=0.3, ly=0.4)
    assert len(cells) == 1 and abs(lens[0] - 0.5) < 1e-13
    cells, lens = O.trace_ray(2, 2, (0.0, 0.0), (1.0, 1.0))
    assert list(cells) == [0, 3] and abs(lens.sum() - math.sqrt(2)) < 1e-13
    with pytest.raises(ValueError):
        O.trace_ray(4, 4, (0.5, 0.5), (0.5, 0.5))
    with pytest.raises(ValueError):
        O.trace_ray(4, 4, (-0.2, 0.5), (1.0, 0.5))


def test_chord_conservation():  # :52-70
    u = O.uniforms(2000, 2024, 0)
    for t in range(1000):
        src, rec = (0.0, u[2 * t]), (1.0, u[2 * t + 1])
        cells, lens = O.trace_ray(59, 55, src, rec)
        chord = math.hypot(1.0, rec[1] - src[1])
        assert abs(lens.sum() - chord) <= 1e-12 * chord
        assert np.all(lens > 0) and np.all(np.diff(cells) != 0)


def test_build_H_rows_and_golden():  # :94-144
    src = [(0.0, (i + 0.5) / 4) for i in range(4)]
    rec = [(1.0, (j + 0.5) / 6) for j in range(6)]
    h = O.build_H(20, 20, src, rec)
    rp, col, val = h.arrays()
    assert h.rows == 24 and h.cols == 400
    for r in range(24):
        assert np.all(np.diff(col[rp[r]:rp[r + 1]]) > 0)  # ascending columns (setFromTriplets)
        chord = math.hypot(1.0, rec[r % 6][1] - src[r // 6][1])
        assert abs(val[rp[r]:rp[r + 1]].sum() - chord) <= 1e-12 * chord
        assert rp[r + 1] - rp[r] <= 40
    D = np.zeros((24, 400))
    for r in range(24):
        D[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    assert np.array_equal(D, GOLD["H_20x20_4x6"])  # bit-identical to the Python transcription
    one = O.build_H(1, 1, [(0.0, 0.4)], [(1.0, 0.6)])
    assert abs(one.arrays()[2][0] - math.sqrt(1.04)) <= 1e-13


# ---------------------------------------------------------------- lowrank.hpp / fast_filter.hpp / uq.hpp
def test_ghep_vs_dense_and_golden():  # test_lowrank.cpp:117-144
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    lam, U, Ub, kept = O.randomized_ghep(p.oracle_cov(), p.oracle_h(), p.sigma2, 24, 20, 19)
    assert len(lam) == 24 and kept == 24 + 20 or kept <= 44
    assert np.all(np.abs(lam - GOLD["ghep_lambda_20x20"]) / GOLD["ghep_lambda_20x20"] < 1e-8)
    gam = p.gamma()
    assert np.linalg.norm(U.T @ np.linalg.solve(gam, U) - np.eye(24)) < 1e-10
    assert rel_err(gam @ Ub, U) < 1e-10


def test_ghep_errors():  # lowrank.hpp:145-151
    p = Problem(5, 5, 2, 2, 1, 2e-4)
    with pytest.raises(ValueError, match="exceeds"):
        O.randomized_ghep(p.oracle_cov(), p.oracle_h(), p.sigma2, 20, 10, 1)
    with pytest.raises(ValueError, match="nonnegative"):
        O.randomized_ghep(p.oracle_cov(), p.oracle_h(), p.sigma2, -1, 10, 1)


def test_offline_reconstruction():  # test_filters.cpp:115-128
    p = Problem(20, 20, 4, 6, 1, 2e-4)
    f = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 24, 20, 5)
    ctx = f.context(gamma_ht=True)
    Hd = csr_dense(p.h)
    A = Hd.T @ Hd / p.sigma2
    gu = np.linalg.solve(p.gamma(), ctx["U"])
    assert np.linalg.norm(gu @ np.diag(ctx["lam"]) @ gu.T - A) <= 1e-8 * np.linalg.norm(A)
    assert rel_err(ctx["gamma_ht"], p.gamma() @ Hd.T) < 1e-11


def test_zero_H_and_first_step():  # test_filters.cpp:130-160
    cov = O.CovarianceOperator(6, 6, **EXPERIMENT)
    h = O.Csr.from_arrays(4, 36, np.zeros(5, np.int32), np.zeros(1, np.int32), np.zeros(1))
    f = O.FastFilter(cov, h, 2e-4, 4, 10, 7)
    assert f.rank == 0
    f.step(np.zeros(4))
    st = f.state()
    assert st["alpha"] == 1.0 and len(st["d"]) == 0 and np.linalg.norm(st["mean"]) == 0.0
    p = Problem(10, 10, 2, 4, 1, 2e-4)
    f = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 8, 20, 9)
    f.step(p.obs[0])
    lam = f.context()["lam"]
    assert np.all(np.abs(f.state()["d"] - lam / (1 + lam)) <= 1e-12 * lam / (1 + lam))


def test_full_rank_matches_dense_kf_golden():  # test_filters.cpp:162-191
    p = Problem(12, 12, 3, 8, 10, 2e-4)
    assert np.array_equal(csr_dense(p.h), GOLD["H_12x12_3x8"])
    assert np.max(np.abs(np.stack(p.obs) - GOLD["kf12_obs"])) < 1e-15
    f = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 24, 20, 11)
    assert f.rank == 24
    gam = p.gamma()
    U = f.context()["U"]
    for k, y in enumerate(p.obs):
        f.step(y)
        st = f.state()
        assert rel_err(st["mean"], GOLD["kf12_means"][k]) < 1e-8
        var = st["alpha"] * 1e-4 - (U ** 2) @ st["d"]
        assert rel_err(var, GOLD["kf12_vars"][k]) < 1e-8
        assert rel_err(f.variance(), var) < 1e-13
        assert st["alpha"] == k + 1 and st["d"].max() < st["alpha"]


def test_uq_kats():  # test_uq.cpp:46-69
    cov = O.CovarianceOperator(5, 5, **EXPERIMENT)
    h = O.build_H(5, 5, [(0.0, 0.5)], [(1.0, 0.5)])
    f = O.FastFilter(cov, h, 2e-4, 1, 4, 3)
    f.set_state(2.0, np.zeros(0), np.zeros(25))
    assert rel_err(f.variance(), np.full(25, 2e-4)) < 1e-14
    assert abs(f.trace_criterion() - 2.0 * 25 * 1e-4) < 1e-17
    f.set_state(1.0, np.zeros(0), np.zeros(25))
    assert f.relative_entropy() == 0.0
    f.set_state(1.0, np.array([0.5]), np.zeros(25))
    assert abs(f.relative_entropy() - (0.5 * math.log(0.5))) < 1e-14
    f.set_state(1.0, np.array([1.0]), np.zeros(25))
    with pytest.raises(RuntimeError):
        f.relative_entropy()


def test_fft_realizations_reproduce_posterior():
    """FFT-mode sampler: E[(x−mean)(x−mean)ᵀ] = αΓ − UDUᵀ."""
    p = Problem(8, 8, 2, 4, 3, 2e-4)
    f = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 8, 20, 3)
    for y in p.obs:
        f.step(y)
    st = f.state()
    ctx = f.context()
    sigma = st["alpha"] * p.gamma() - ctx["U"] @ np.diag(st["d"]) @ ctx["U"].T
    draws = 4000
    acc = np.zeros((64, 64))
    for s in range(0, draws, 8):
        X = f.realizations(1000 + s, 8) - st["mean"][:, None]
        acc += X @ X.T
    emp = acc / draws
    assert np.linalg.norm(emp - sigma) <= 0.1 * np.linalg.norm(sigma)
    assert abs(np.trace(emp) - f.trace_criterion()) <= 0.05 * f.trace_criterion()
