"""Python mirror of the reference's ``namespace fastkf`` hot-path API, over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/fastkf
(``std::invalid_argument`` → ValueError, ``std::runtime_error`` → RuntimeError), so the
parity tests read like the reference's Catch2 suites.  Every numeric call runs the
sm_100a kernels in libfastkf_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from ._native import DeviceArray, DomainError, check, lib, ptr

POWERED_EXPONENTIAL = 0
MATERN = 1


@dataclasses.dataclass(frozen=True)
class Grid:  # grid.hpp:22-63
    nx: int
    ny: int
    lx: float = 1.0
    ly: float = 1.0

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError(f"grid: nx and ny must be positive, got {self.nx}x{self.ny}")
        if not (self.lx > 0.0 and self.ly > 0.0):
            raise ValueError("grid: domain lengths must be positive")

    def size(self) -> int:
        return self.nx * self.ny

    def dx(self):
        return self.lx / self.nx

    def dy(self):
        return self.ly / self.ny

    def index(self, ix, iy):
        return ix * self.ny + iy


@dataclasses.dataclass(frozen=True)
class KernelSpec:  # kernel.hpp:19-48
    family: int = POWERED_EXPONENTIAL
    theta: float = 1.0
    length: float = 0.2
    power: float = 1.0
    nu: float = 0.5
    alpha_scale: float = 0.0

    def args(self):
        return (self.family, self.theta, self.length, self.power, self.nu, self.alpha_scale)


def kernel_eval(spec: KernelSpec, r: float) -> float:  # kernel.hpp:51-63
    out = C.c_double()
    check(lib().fkb_kernel_eval(*spec.args(), float(r), C.byref(out)))
    return out.value


def next_smooth(n: int) -> int:  # covariance.hpp:35-43
    return int(lib().fkb_next_smooth(int(n)))


# ------------------------------------------------------------------ tomography.hpp
def trace_ray(grid: Grid, src, rec):
    """tomography.hpp:29-86 → (cells, lengths) in traversal order."""
    cap = 4 * (grid.nx + grid.ny) + 8
    cells = np.empty(cap, dtype=np.int64)
    lens = np.empty(cap)
    cnt = C.c_int()
    check(lib().fkb_trace_ray(grid.nx, grid.ny, grid.lx, grid.ly, float(src[0]), float(src[1]), float(rec[0]),
                              float(rec[1]), cap, cells, lens, C.byref(cnt)))
    return cells[:cnt.value].copy(), lens[:cnt.value].copy()


@dataclasses.dataclass
class SourceReceiverLayout:  # tomography.hpp:90-126
    sources: np.ndarray
    receivers: np.ndarray

    @staticmethod
    def cross_well(grid: Grid, n_sou: int, n_rec: int, source_x: float = 0.0, receiver_x: float = -1.0):
        if n_sou < 1 or n_rec < 1:
            raise ValueError("layout: n_sou and n_rec must be positive")
        if receiver_x < 0.0:
            receiver_x = grid.lx
        s = np.array([[source_x, (i + 0.5) * grid.ly / n_sou] for i in range(n_sou)])
        r = np.array([[receiver_x, (j + 0.5) * grid.ly / n_rec] for j in range(n_rec)])
        return SourceReceiverLayout(s, r)

    def n_m(self):
        return len(self.sources) * len(self.receivers)


@dataclasses.dataclass
class CsrMatrix:  # SparseRowMatrix (grid.hpp:15)
    rows: int
    cols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self):
        return len(self.val)

    def matvec(self, x):
        out = np.zeros(self.rows)
        for r in range(self.rows):
            a, b = self.rowptr[r], self.rowptr[r + 1]
            out[r] = np.dot(self.val[a:b], x[self.col[a:b]])
        return out

    def scale_rows(self, s):
        rows = np.repeat(np.arange(self.rows), np.diff(self.rowptr))
        return CsrMatrix(self.rows, self.cols, self.rowptr, self.col, self.val / np.asarray(s)[rows])

    @staticmethod
    def vstack(mats):
        rp = [mats[0].rowptr]
        off = mats[0].rowptr[-1]
        for m in mats[1:]:
            rp.append(m.rowptr[1:] + off)
            off += m.rowptr[-1]
        return CsrMatrix(sum(m.rows for m in mats), mats[0].cols, np.concatenate(rp).astype(np.int32),
                         np.concatenate([m.col for m in mats]).astype(np.int32),
                         np.concatenate([m.val for m in mats]))


def build_H(grid: Grid, layout: SourceReceiverLayout) -> CsrMatrix:  # tomography.hpp:130-146
    s = np.ascontiguousarray(np.asarray(layout.sources, dtype=np.float64).reshape(-1, 2)).ravel()
    r = np.ascontiguousarray(np.asarray(layout.receivers, dtype=np.float64).reshape(-1, 2)).ravel()
    rows, nnz = C.c_int(), C.c_longlong()
    L = lib()
    check(L.fkb_build_H(grid.nx, grid.ny, grid.lx, grid.ly, len(s) // 2, s, len(r) // 2, r, C.byref(rows),
                        C.byref(nnz), None, None, None, 0))
    rowptr = np.empty(rows.value + 1, dtype=np.int32)
    col = np.empty(max(nnz.value, 1), dtype=np.int32)
    val = np.empty(max(nnz.value, 1))
    check(L.fkb_build_H(grid.nx, grid.ny, grid.lx, grid.ly, len(s) // 2, s, len(r) // 2, r, C.byref(rows),
                        C.byref(nnz), ptr(rowptr), ptr(col), ptr(val), nnz.value))
    return CsrMatrix(rows.value, grid.size(), rowptr, col[:nnz.value], val[:nnz.value])


def sym_eig(a: np.ndarray):
    """Host symmetric eigensolver used inside the GHEP (ascending; SelfAdjointEigenSolver stand-in)."""
    n = a.shape[0]
    A = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).ravel()
    w = np.empty(n)
    Z = np.empty(n * n)
    check(lib().fkb_sym_eig(n, A, w, Z))
    return w, Z.reshape(n, n).T


def sym_eig_device(a: np.ndarray):
    """The same on the GPU (block Jacobi, eig.cu): (ascending eigenvalues, eigenvectors, sweeps)."""
    n = a.shape[0]
    A = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).ravel()
    w = np.empty(n)
    Z = np.empty(n * n)
    sw = C.c_int()
    check(lib().fkb_sym_eig_device(n, A, w, Z, C.byref(sw)))
    return w, Z.reshape(n, n).T, sw.value


def sym_eig_tridiag(a: np.ndarray):
    """GPU Householder tridiagonalization + QL (tdeig.cu): (ascending eigenvalues, eigenvectors)."""
    n = a.shape[0]
    A = np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).ravel()
    w = np.empty(n)
    Z = np.empty(n * n)
    check(lib().fkb_sym_eig_tridiag(n, A, w, Z))
    return w, Z.reshape(n, n).T


# ------------------------------------------------------------------ covariance.hpp (FFT mode)
class CovarianceOperator:
    """CovarianceOperator(grid, spec, CovMode::fft) — covariance.hpp:69-353 on the GPU."""

    def __init__(self, grid: Grid, spec: KernelSpec):
        self.grid = grid
        self.spec = spec
        h = C.c_void_p()
        check(lib().fkb_cov_create(grid.nx, grid.ny, grid.lx, grid.ly, *spec.args(), C.byref(h)))
        self._h = h
        mx, my = C.c_int(), C.c_int()
        check(lib().fkb_cov_dims(self._h, C.byref(mx), C.byref(my)))
        self.mx, self.my = mx.value, my.value

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().fkb_cov_destroy(self._h)
            self._h = None

    def size(self) -> int:
        return self.grid.size()

    def spectrum(self) -> np.ndarray:
        out = np.empty(self.mx * self.my)
        check(lib().fkb_cov_spectrum(self._h, out))
        return out

    def apply_count(self) -> int:
        return int(lib().fkb_cov_apply_count(self._h))

    def diagonal(self):  # covariance.hpp:178
        return np.full(self.size(), self.spec.theta)

    def trace(self):  # covariance.hpp:180
        return float(self.size()) * self.spec.theta

    def apply(self, x) -> np.ndarray:
        """Γx for a vector or column-wise for an N×c matrix (covariance.hpp:101-115)."""
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        X = x.reshape(-1, 1) if vec else x
        n = self.size()
        if X.shape[0] != n:
            raise ValueError(f"cov_apply: expected vector of length {n}, got {X.shape[0]}")
        Xf = np.ascontiguousarray(X.T)  # column j contiguous
        Y = np.empty_like(Xf)
        check(lib().fkb_cov_apply(self._h, ptr(Xf), n, X.shape[1], ptr(Y), n))
        return Y[0].copy() if vec else np.asfortranarray(Y.T)

    def apply_device(self, dX, ldx, ncols, dY, ldy):
        check(lib().fkb_cov_apply_device(self._h, dX, ldx, ncols, dY, ldy))

    def sample_pair(self, seed: int, stream: int = 0):  # covariance.hpp:190-197
        a = np.empty(self.size())
        b = np.empty(self.size())
        check(lib().fkb_cov_sample_pair(self._h, seed, stream, a, b))
        return a, b

    def sample(self, seed: int, stream: int = 0):
        return self.sample_pair(seed, stream)[0]

    @property
    def stream(self):
        return lib().fkb_cov_stream(self._h)


def gaussian_matrix(rows: int, cols: int, seed: int, base_stream: int = 0) -> np.ndarray:
    """rng.hpp:79-86 generated by the device RNG (column-major result)."""
    out = np.empty(rows * cols)
    check(lib().fkb_gaussian_matrix(rows, cols, seed, base_stream, out))
    return out.reshape(cols, rows).T


# ------------------------------------------------------------------ fast_filter.hpp / uq.hpp
class FkfContext:
    """fkf_init (fast_filter.hpp:51-75) + the device-resident LowRankState (:21-37).

    The state lives on the GPU and W ≡ U (constant-H regime); ``state()`` downloads it.
    """

    def __init__(self, cov: CovarianceOperator, h: CsrMatrix, sigma2: float, k_rank: int, p_oversample: int,
                 seed: int):
        self.cov = cov
        self.h = h
        self.sigma2 = float(sigma2)
        f = C.c_void_p()
        check(lib().fkb_fkf_init(cov._h, h.rows, h.cols, np.ascontiguousarray(h.rowptr, np.int32),
                                 np.ascontiguousarray(h.col if len(h.col) else np.zeros(1, np.int32), np.int32),
                                 np.ascontiguousarray(h.val if len(h.val) else np.zeros(1), np.float64),
                                 self.sigma2, int(k_rank), int(p_oversample), int(seed), C.byref(f)))
        self._f = f
        r, kept = C.c_int(), C.c_int()
        check(lib().fkb_filter_rank(self._f, C.byref(r), C.byref(kept)))
        self.r, self.kept_cols = r.value, kept.value
        self.n, self.m = cov.size(), h.rows

    def __del__(self):
        if getattr(self, "_f", None) and self._f.value:
            lib().fkb_filter_destroy(self._f)
            self._f = None

    def rank(self):
        return self.r

    @property
    def lam(self) -> np.ndarray:
        out = np.empty(max(self.r, 1))
        check(lib().fkb_filter_lambda(self._f, out))
        return out[: self.r]

    def _get(self, which, rows, cols):
        out = np.empty(max(rows * cols, 1))
        check(lib().fkb_filter_get(self._f, which, out))
        return out[: rows * cols].reshape(cols, rows).T

    def U(self):
        return self._get(0, self.n, self.r)

    def Ubar(self):
        return self._get(1, self.n, self.r)

    def h_gamma_ht(self):
        return self._get(2, self.m, self.m)

    def h_u(self):
        return self._get(3, self.m, self.r)

    # -- state
    def step(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        check(lib().fkb_fkf_step(self._f, ptr(y), len(y)))

    def run(self, ys, count=None, seed=0):
        """len(ys) steps in one call with every step's new state (fkb_fkf_run; with count: the fused
        diag Σ and `count` realizations too, fkb_fkf_run_uq).  Returns dict(alpha (n,), d (n, r),
        mean (n, N)[, var (n, N), x (n, count, N)])."""
        Y = np.ascontiguousarray(np.atleast_2d(np.asarray(ys, dtype=np.float64)))
        ns = Y.shape[0]
        r = max(self.r, 1)
        al, d, mean = np.zeros(max(ns, 1)), np.zeros((max(ns, 1), r)), np.zeros((max(ns, 1), self.n))
        if count is None:
            check(lib().fkb_fkf_run(self._f, ptr(Y), ns, Y.shape[1], ptr(al), ptr(d), r, ptr(mean), self.n))
            return dict(alpha=al[:ns], d=d[:ns, : self.r], mean=mean[:ns])
        x, var = np.zeros((max(ns, 1), max(count, 1), self.n)), np.zeros((max(ns, 1), self.n))
        check(lib().fkb_fkf_run_uq(self._f, ptr(Y), ns, Y.shape[1], int(seed), int(count), ptr(x), ptr(var), ptr(al),
                                   ptr(d), r, ptr(mean), self.n))
        return dict(alpha=al[:ns], d=d[:ns, : self.r], mean=mean[:ns], var=var[:ns], x=x[:ns, :count])

    def step_device(self, d_y):
        check(lib().fkb_fkf_step_device(self._f, d_y))

    def step_uq(self, y, seed: int, count: int):
        """One step + diag Σ and `count` realizations of the new state from one fused U pass
        (fkf_step + variance + RealizationPropagator::at, uq.hpp:16-112).  Returns
        (state dict, realizations N×count, variance)."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        x, var = np.empty(max(self.n * count, 1)), np.empty(self.n)
        a = C.c_double()
        d, mean = np.empty(max(self.r, 1)), np.empty(self.n)
        check(lib().fkb_fkf_step_uq(self._f, ptr(y), len(y), int(seed), int(count), ptr(x), ptr(var), C.byref(a), ptr(d),
                                    ptr(mean)))
        st = self.state()
        return st, x[: self.n * count].reshape(count, self.n).T.copy(), var

    def step_uq_device(self, d_y, seed, count, d_x, d_var):
        check(lib().fkb_fkf_step_uq_device(self._f, d_y, int(seed), int(count), d_x, d_var))

    def steps_async(self, d_ys, nsteps, ldy):
        check(lib().fkb_fkf_steps_async(self._f, d_ys, nsteps, ldy))

    def sync(self, nsteps):
        check(lib().fkb_fkf_sync(self._f, nsteps))

    def state(self):
        a, st, rk = C.c_double(), C.c_int(), C.c_int()
        d = np.empty(max(self.r, 1))
        mean = np.empty(self.n)
        check(lib().fkb_filter_state(self._f, C.byref(a), C.byref(st), C.byref(rk), ptr(d), ptr(mean)))
        return dict(alpha=a.value, step=st.value, rank=rk.value, d=d[: rk.value].copy(), mean=mean)

    def set_state(self, alpha, d, mean, step=0):
        d = np.ascontiguousarray(d, dtype=np.float64)
        mean = np.ascontiguousarray(mean, dtype=np.float64)
        check(lib().fkb_filter_set_state(self._f, float(alpha), int(step), len(d), ptr(d) if len(d) else None,
                                         ptr(mean)))

    def reset(self):
        check(lib().fkb_filter_reset(self._f))

    def ghep_residual(self):
        """lowrank.hpp:215-228 for the context's GEP (Γ⁻¹U from Ū, no CG)."""
        out = np.empty(max(self.r, 1))
        check(lib().fkb_filter_ghep_residual(self._f, out))
        return out[: self.r]

    # -- UQ
    def variance(self):
        out = np.empty(self.n)
        check(lib().fkb_variance(self._f, out))
        return out

    def trace_criterion(self):
        v = C.c_double()
        check(lib().fkb_trace_criterion(self._f, C.byref(v)))
        return v.value

    def relative_entropy(self):
        v = C.c_double()
        check(lib().fkb_relative_entropy(self._f, C.byref(v)))
        return v.value

    def realizations(self, seed: int, count: int):
        out = np.empty(max(self.n * count, 1))
        check(lib().fkb_realizations(self._f, seed, count, out))
        return out[: self.n * count].reshape(count, self.n).T

    def realizations_device(self, seed, count, d_out, d_var=None):
        check(lib().fkb_realizations_device(self._f, seed, count, d_out, d_var))

    def variance_device(self, d_out):
        check(lib().fkb_variance_device(self._f, d_out))

    def spmm_device(self, trans, dX, ldx, ncols, dY, ldy):
        check(lib().fkb_filter_spmm(self._f, trans, dX, ldx, ncols, dY, ldy))

    def spmm_rm_device(self, trans, dX, ncols, dY):
        """Y = H X (trans 0) / Hᵀ X (trans 1) on row-major device blocks."""
        check(lib().fkb_filter_spmm_rm(self._f, trans, dX, ncols, dY))

    @property
    def stream(self):
        return lib().fkb_filter_stream(self._f)

    def launches_per_step(self):
        return int(lib().fkb_filter_launches_per_step(self._f))

    def set_solver(self, mode: int):
        """1 (default): Woodbury solve in G's eigenbasis; 0: reference-order m×m LLT."""
        check(lib().fkb_filter_set_solver(self._f, int(mode)))

    def eig_sweeps(self) -> int:
        return int(lib().fkb_filter_eig_sweeps(self._f))

    def set_pcg_maxit(self, maxit: int):
        """Iteration cap of the capacitance PCG; 0 forces the exact Cholesky fallback."""
        check(lib().fkb_filter_set_pcg_maxit(self._f, int(maxit)))

    def cap_stats(self):
        """(PCG iterations, Cholesky fallback used) of the last step's capacitance solve."""
        it, fb = C.c_int(), C.c_int()
        check(lib().fkb_filter_cap_stats(self._f, C.byref(it), C.byref(fb)))
        return it.value, bool(fb.value)

    def g_eig(self):
        th = np.empty(max(self.m, 1))
        Pm = np.empty(max(self.m * self.m, 1))
        check(lib().fkb_filter_get_eig(self._f, ptr(th), ptr(Pm)))
        return th[: self.m], Pm[: self.m * self.m].reshape(self.m, self.m).T

    def phase_times(self, reps: int = 3):
        """Runs `reps` real steps (advancing the state) with CUDA events per phase."""
        ms = np.zeros(32)
        names = C.create_string_buffer(1024)
        cnt = C.c_int()
        check(lib().fkb_filter_phase_times(self._f, int(reps), ms, names, 1024, C.byref(cnt)))
        keys = names.value.decode().split(",") if cnt.value else []
        return dict(zip(keys, ms[: cnt.value].tolist()))


    def graph_timing(self, on: bool = True):
        """Re-captures the step graph with timing events at every phase boundary."""
        check(lib().fkb_filter_graph_timing(self._f, 1 if on else 0))

    def graph_phase_times(self):
        """Per-phase device ms of the last graph replay (needs graph_timing(True))."""
        ms = np.zeros(64)
        names = C.create_string_buffer(2048)
        cnt = C.c_int()
        check(lib().fkb_filter_graph_phase_times(self._f, ms, names, 2048, C.byref(cnt)))
        keys = names.value.decode().split(",") if cnt.value else []
        return dict(zip(keys, ms[: cnt.value].tolist()))


@dataclasses.dataclass
class FekfOptions:  # fast_filter.hpp:127-134
    k_rank: int = -1  # −1: n_m
    oversampling: int = 20
    trunc_tol: float = 1e-5
    relinearizations: int = 1
    seed: int = 0


@dataclasses.dataclass(frozen=True)
class BoxCox:  # boxcox.hpp:14-17 (the maps run on the device inside fekf_step)
    alpha: float = 1.0


class ExtendedFilter:
    """fekf_step (fast_filter.hpp:127-224) on a device-resident LowRankState.

    Binds Γ (``cov``) and the ray operator ``h`` once (every reference caller keeps them
    fixed across steps, driver.hpp:305-333); ``reset(mean0)`` is zero_start with the
    initial mean of driver.hpp:315-316.  Besides W the state carries W̄ = Γ⁻¹W.
    """

    def __init__(self, cov: CovarianceOperator, h: CsrMatrix, mean0=None):
        self.cov, self.h = cov, h
        self.n, self.m = cov.size(), h.rows
        e = C.c_void_p()
        check(lib().fkb_ekf_create(cov._h, h.rows, h.cols, np.ascontiguousarray(h.rowptr, np.int32),
                                   np.ascontiguousarray(h.col if len(h.col) else np.zeros(1, np.int32), np.int32),
                                   np.ascontiguousarray(h.val if len(h.val) else np.zeros(1), np.float64),
                                   C.byref(e)))
        self._e = e
        if mean0 is not None:
            self.reset(mean0)

    def __del__(self):
        if getattr(self, "_e", None) and self._e.value:
            lib().fkb_ekf_destroy(self._e)
            self._e = None

    def reset(self, mean0):
        check(lib().fkb_ekf_reset(self._e, np.ascontiguousarray(np.broadcast_to(mean0, (self.n,)), np.float64)))

    def step(self, y, sigma2: float, transform: BoxCox, opts: FekfOptions = FekfOptions()):
        y = np.ascontiguousarray(y, np.float64)
        check(lib().fkb_ekf_step(self._e, y, y.size, float(sigma2), float(transform.alpha), int(opts.k_rank),
                                 int(opts.oversampling), float(opts.trunc_tol), int(opts.relinearizations),
                                 int(opts.seed)))

    def rank(self) -> int:
        r = C.c_int()
        check(lib().fkb_ekf_state(self._e, None, None, C.byref(r)))
        return r.value

    def state(self, with_w: bool = True):
        a, st, r = C.c_double(), C.c_int(), C.c_int()
        check(lib().fkb_ekf_state(self._e, C.byref(a), C.byref(st), C.byref(r)))
        n, k = self.n, r.value
        mean, d = np.empty(n), np.empty(k)
        w = np.empty((k, n)) if with_w else None
        wb = np.empty((k, n)) if with_w else None
        check(lib().fkb_ekf_read(self._e, ptr(mean), ptr(d) if k else None, ptr(w) if with_w and k else None,
                                 ptr(wb) if with_w and k else None))
        out = {"alpha": a.value, "step": st.value, "mean": mean, "d": d}
        if with_w:
            out["w"] = w.T if k else np.zeros((n, 0))
            out["wbar"] = wb.T if k else np.zeros((n, 0))
        return out

    def trace_criterion(self) -> float:  # uq.hpp:25-34
        t = C.c_double()
        check(lib().fkb_ekf_uq(self._e, C.byref(t), None))
        return t.value

    def relative_entropy(self) -> float:  # uq.hpp:36-53
        h = C.c_double()
        check(lib().fkb_ekf_uq(self._e, None, C.byref(h)))
        return h.value

    def last_step_info(self):
        g, sw = C.c_int(), C.c_int()
        check(lib().fkb_ekf_last(self._e, C.byref(g), C.byref(sw)))
        return {"gep_rank": g.value, "sweeps": sw.value}


def fekf_step(filt: ExtendedFilter, y, sigma2, transform: BoxCox, opts: FekfOptions = FekfOptions()):
    """Advances the extended filter's device state by one cycle (fast_filter.hpp:142-224)."""
    filt.step(y, sigma2, transform, opts)
    return filt.state()


class Ensemble:
    """Ensemble (enkf.hpp:15-28) resident on the GPU and bound to Γ and H: ``enkf_init``
    (:30-34) at construction, ``step`` = enkf_step (:49-94)."""

    def __init__(self, cov: CovarianceOperator, h: CsrMatrix, n_members: int):
        self.cov, self.h = cov, h
        self.n, self.m, self.n_members = cov.size(), h.rows, int(n_members)
        e = C.c_void_p()
        check(lib().fkb_enkf_init(cov._h, h.rows, h.cols, np.ascontiguousarray(h.rowptr, np.int32),
                                  np.ascontiguousarray(h.col if len(h.col) else np.zeros(1, np.int32), np.int32),
                                  np.ascontiguousarray(h.val if len(h.val) else np.zeros(1), np.float64),
                                  self.n_members, C.byref(e)))
        self._e = e

    def __del__(self):
        if getattr(self, "_e", None) and self._e.value:
            lib().fkb_enkf_destroy(self._e)
            self._e = None

    def size(self) -> int:
        return self.n_members

    def step(self, y, sigma2: float, seed: int):
        y = np.ascontiguousarray(y, np.float64)
        check(lib().fkb_enkf_step(self._e, y, y.size, float(sigma2), int(seed)))

    @property
    def members(self) -> np.ndarray:  # n × N_e
        out = np.empty(self.n * self.n_members)
        check(lib().fkb_enkf_members(self._e, out))
        return out.reshape(self.n_members, self.n).T

    @members.setter
    def members(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n, self.n_members):
            raise ValueError("ensemble: members must be n × N_e")
        check(lib().fkb_enkf_set_members(self._e, np.ascontiguousarray(x.T).ravel()))

    def mean(self) -> np.ndarray:
        out = np.empty(self.n)
        check(lib().fkb_enkf_mean(self._e, out))
        return out

    def covariance(self) -> np.ndarray:  # enkf.hpp:22-25 (host; desk scale)
        x = self.members
        dev = x - x.mean(axis=1, keepdims=True)
        return dev @ dev.T / (self.n_members - 1)


def enkf_init(cov, h, n_members) -> Ensemble:
    return Ensemble(cov, h, n_members)


def enkf_step(ens: Ensemble, y, sigma2, seed) -> Ensemble:
    """Advances the device ensemble by one cycle (enkf.hpp:49-94)."""
    ens.step(y, sigma2, seed)
    return ens


# ------------------------------------------------------------------ field_io.hpp (FKF1 / FKS1)
def write_field(path, nx: int, ny: int, data) -> None:
    """write_field (field_io.hpp:66-79): "FKF1", uint32 nx, uint32 ny, float64 x-major."""
    data = np.ascontiguousarray(data, dtype="<f8")
    if data.size != nx * ny:
        raise ValueError(f"write_field: data length does not match {nx}x{ny}")
    with open(path, "wb") as f:
        f.write(b"FKF1" + np.array([nx, ny], dtype="<u4").tobytes() + data.tobytes())


def read_field(path):
    """read_field (field_io.hpp:81-95) → (nx, ny, data)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"FKF1":
        raise RuntimeError(f"not a FKF1 field file: {path}")
    if len(raw) < 12:
        raise RuntimeError(f"truncated file: {path}")
    nx, ny = (int(v) for v in np.frombuffer(raw, "<u4", 2, 4))
    if nx < 1 or ny < 1 or nx * ny > (1 << 31):
        raise RuntimeError(f"implausible field dimensions in {path}")
    if len(raw) < 12 + 8 * nx * ny:
        raise RuntimeError(f"truncated file: {path}")
    return nx, ny, np.frombuffer(raw, "<f8", nx * ny, 12).copy()


def write_state(path, state: dict, w=None) -> None:
    """write_state (field_io.hpp:100-113): "FKS1", uint32 n, r, step, float64 α, mean, D, W
    (column-major).  ``w`` defaults to state["w"]; for an FkfContext state pass ctx.u()."""
    mean = np.ascontiguousarray(state["mean"], "<f8")
    d = np.ascontiguousarray(state["d"], "<f8")
    w = np.asarray(state["w"] if w is None else w, dtype=np.float64)
    if w.shape != (mean.size, d.size):
        raise ValueError("write_state: W does not match the state")
    with open(path, "wb") as f:
        f.write(b"FKS1" + np.array([mean.size, d.size, int(state["step"])], "<u4").tobytes()
                + np.array([state["alpha"]], "<f8").tobytes() + mean.tobytes() + d.tobytes()
                + np.asfortranarray(w).astype("<f8").tobytes(order="F"))


def read_state(path) -> dict:
    """read_state (field_io.hpp:115-135) → {"alpha", "step", "mean", "d", "w"}."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"FKS1":
        raise RuntimeError(f"not a FKS1 state file: {path}")
    if len(raw) < 24:
        raise RuntimeError(f"truncated file: {path}")
    n, r, step = (int(v) for v in np.frombuffer(raw, "<u4", 3, 4))
    alpha = float(np.frombuffer(raw, "<f8", 1, 16)[0])
    need = 24 + 8 * (n + r + n * r)
    if len(raw) < need:
        raise RuntimeError(f"truncated file: {path}")
    vals = np.frombuffer(raw, "<f8", n + r + n * r, 24)
    return {"alpha": alpha, "step": step, "mean": vals[:n].copy(), "d": vals[n:n + r].copy(),
            "w": vals[n + r:].reshape(r, n).T.copy()}


def fkf_init(cov, h, sigma2, k_rank, p_oversample, seed) -> FkfContext:
    return FkfContext(cov, h, sigma2, k_rank, p_oversample, seed)


def fkf_step(ctx: FkfContext, y):
    """Advances ctx's device state by one cycle (fast_filter.hpp:84-125)."""
    ctx.step(y)
    return ctx.state()


def variance(ctx: FkfContext):
    return ctx.variance()


def trace_criterion(ctx: FkfContext):
    return ctx.trace_criterion()


def relative_entropy(ctx: FkfContext):
    return ctx.relative_entropy()


__all__ = ["Grid", "KernelSpec", "kernel_eval", "next_smooth", "trace_ray", "SourceReceiverLayout", "CsrMatrix",
           "build_H", "sym_eig", "sym_eig_device", "CovarianceOperator", "gaussian_matrix", "FkfContext", "fkf_init", "fkf_step",
           "variance", "trace_criterion", "relative_entropy", "DeviceArray", "POWERED_EXPONENTIAL", "MATERN",
           "FekfOptions", "BoxCox", "ExtendedFilter", "fekf_step", "DomainError", "Ensemble", "enkf_init",
           "enkf_step", "write_field",
           "read_field", "write_state", "read_state"]
