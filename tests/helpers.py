"""Shared test fixtures: desk-scale problems restated from the reference's Catch2 suites
(proj/tests/test_filters.cpp:36-52, test_uq.cpp:28-44) and dense numpy oracles
(proj/tests/oracles.hpp:35-108).  Inputs are generated once and fed identically to the
product (paper_1405_2276_b200) and to the CPU oracle (oracle/)."""
from __future__ import annotations

import math

import numpy as np

from paper_1405_2276_b200 import workloads as W


def rel_err(got, want):  # oracles.hpp:75-85
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def centers(nx, ny, lx=1.0, ly=1.0):
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    return ((ix + 0.5) * (lx / nx)).ravel(), ((iy + 0.5) * (ly / ny)).ravel()


def kernel_fn(family, theta, length, power=1.0, nu=0.5, alpha_scale=0.0):
    from scipy.special import gamma, kv

    def f(r):
        r = np.asarray(r, dtype=np.float64)
        if family == 0:
            v = theta * np.exp(-np.power(r / length, power))
        else:
            sc = alpha_scale if alpha_scale > 0 else 1.0 / length
            a = math.sqrt(2.0 * nu) * sc * r
            with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
                v = theta * 2.0 ** (1 - nu) / gamma(nu) * a ** nu * kv(nu, a)
            v = np.where(a > 700.0, 0.0, v)
        return np.where(r == 0.0, theta, v)
    return f


def kernel_matrix(nx, ny, f, lx=1.0, ly=1.0):  # oracles.hpp:35-44
    cx, cy = centers(nx, ny, lx, ly)
    r = np.sqrt((cx[:, None] - cx[None, :]) ** 2 + (cy[:, None] - cy[None, :]) ** 2)
    return f(r)


def sym_sqrt(a):  # oracles.hpp:47-52
    w, v = np.linalg.eigh(a)
    return (v * np.sqrt(np.maximum(w, 0.0))) @ v.T


def dense_ghep(a, gamma):  # oracles.hpp:61-73
    root = sym_sqrt(gamma)
    w, v = np.linalg.eigh(root @ a @ root)
    return w[::-1], root @ v[:, ::-1]


def plume_field(nx, ny, t_hours, center=(0.5, 0.5), sigma=(0.1, 0.1), rate=1e-5, max_pert=5e-3):
    """PlumeModel default blob (tomography.hpp:148-195)."""
    cx, cy = centers(nx, ny)
    amp = rate * t_hours
    if amp == 0.0:
        return np.zeros(nx * ny)
    ex = (cx - center[0]) / sigma[0]
    ey = (cy - center[1]) / sigma[1]
    return np.minimum(amp * np.exp(-0.5 * (ex * ex + ey * ey)), max_pert)


def simulate_observations(h, s, sigma2, seed, stream=0):  # tomography.hpp:198-211
    y = W.csr_matvec(h.rowptr, h.col, h.val, s)
    if sigma2 > 0.0:
        y = y + math.sqrt(sigma2) * W.rng_normals(h.rows, seed, stream)
    return y


EXPERIMENT = dict(family=0, theta=1e-4, length=0.2, power=0.5)  # test_filters.cpp:19-25


class Problem:
    """test_filters.cpp:36-52: grid, cross-well H, plume observations at t = 3k hours."""

    def __init__(self, nx, ny, n_sou, n_rec, n_steps, sigma2, kernel=EXPERIMENT, obs_seed=77):
        import paper_1405_2276_b200 as P
        self.nx, self.ny = nx, ny
        self.grid = P.Grid(nx, ny)
        self.kernel = dict(kernel)
        self.layout = P.SourceReceiverLayout.cross_well(self.grid, n_sou, n_rec)
        self.h = P.build_H(self.grid, self.layout)
        self.sigma2 = sigma2
        self.obs = [simulate_observations(self.h, plume_field(nx, ny, 3.0 * k), sigma2, W.derive_seed(obs_seed, k))
                    for k in range(1, n_steps + 1)]

    def spec(self):
        import paper_1405_2276_b200 as P
        return P.KernelSpec(**self.kernel)

    def gamma(self):
        return kernel_matrix(self.nx, self.ny, kernel_fn(**self.kernel))

    def oracle_cov(self):
        from oracle import oracle as O
        return O.CovarianceOperator(self.nx, self.ny, **self.kernel)

    def oracle_h(self):
        from oracle import oracle as O
        return O.Csr.from_arrays(self.h.rows, self.h.cols, self.h.rowptr, self.h.col, self.h.val)


def dense_kf(gamma, h_dense, obs, sigma2):
    """dense_kf_step (dense_filter.hpp:41-62) restated in numpy, zero start."""
    n = gamma.shape[0]
    mean = np.zeros(n)
    cov = np.zeros((n, n))
    out = []
    for y in obs:
        p = cov + gamma
        s = h_dense @ p @ h_dense.T + sigma2 * np.eye(h_dense.shape[0])
        k = np.linalg.solve(s, h_dense @ p).T
        mean = mean + k @ (y - h_dense @ mean)
        cov = p - k @ h_dense @ p
        out.append((mean.copy(), cov.copy()))
    return out


def csr_dense(h):
    A = np.zeros((h.rows, h.cols))
    for r in range(h.rows):
        a, b = h.rowptr[r], h.rowptr[r + 1]
        A[r, h.col[a:b]] = h.val[a:b]
    return A


def workload_inputs(name, steps=None):
    """BASELINE config inputs: (workload, H CsrMatrix (whitened for c3), ys, sigma2)."""
    return W.problem(name, steps)


def boxcox_np(alpha, x, which):
    """BoxCox (boxcox.hpp:25-50) restated in numpy (no domain checks)."""
    x = np.asarray(x, dtype=np.float64)
    if alpha == 1.0:
        return {"forward": x - 1.0, "inverse": x + 1.0, "derivative": np.ones_like(x)}[which]
    if which == "forward":
        return alpha * (np.power(x, 1.0 / alpha) - 1.0)
    base = (x + alpha) / alpha
    return np.power(base, alpha) if which == "inverse" else np.power(base, alpha - 1.0)


def dense_ekf(gamma, h_dense, obs, sigma2, bc_alpha, mean0, relinearizations=1):
    """dense_ekf_step (dense_filter.hpp:68-106) restated in numpy, zero start with mean0."""
    n = gamma.shape[0]
    mean = np.array(mean0, dtype=np.float64)
    cov = np.zeros((n, n))
    out = []
    for y in obs:
        pred = cov + gamma
        eta = mean.copy()
        for _ in range(relinearizations):
            hk = h_dense * boxcox_np(bc_alpha, eta, "derivative")[None, :]
            h_eta = h_dense @ boxcox_np(bc_alpha, eta, "inverse")
            hp = hk @ pred
            s = hp @ hk.T + sigma2 * np.eye(hk.shape[0])
            s = 0.5 * (s + s.T)
            resid = y - h_eta - hk @ (mean - eta)
            eta_next = mean + hp.T @ np.linalg.solve(s, resid)
            change = np.linalg.norm(eta_next - eta)
            eta = eta_next
            if change <= 1e-6 * np.linalg.norm(eta):
                break
        mean = eta
        cov = pred - hp.T @ np.linalg.solve(s, hp)
        cov = 0.5 * (cov + cov.T)
        out.append((mean.copy(), cov.copy()))
    return out


def low_rank_cov(alpha, w, d, gamma):  # oracles.hpp: Σ = αΓ − W·diag(d)·Wᵀ
    return alpha * gamma - (w * d[None, :]) @ w.T
