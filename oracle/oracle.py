"""ctypes binding for the CPU restatement oracle (oracle/fastkf_oracle.cpp).

TEST INFRASTRUCTURE ONLY — the parity checker.  Only tests/, the smoke() check in
__graft_entry__.py and bench.py's cpu_baseline / ``--impl reference`` legs may import
this module.  The product package ``paper_1405_2276_b200`` never imports it.

Each wrapper names the reference function it restates (file:line under
/root/reference/proj/include/fastkf/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_d = C.c_double
_i = C.c_int
_ll = C.c_longlong
_u64 = C.c_uint64
_p = C.c_void_p
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_llp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_set_threads": (None, [_i]),
        "orc_max_threads": (_i, []),
        "orc_splitmix64": (_u64, [_u64]),
        "orc_derive_seed": (_u64, [_u64, _u64]),
        "orc_gaussian_vector": (None, [_ll, _u64, _u64, _dp]),
        "orc_gaussian_matrix": (None, [_ll, _ll, _u64, _u64, _dp]),
        "orc_uniforms": (None, [_ll, _u64, _u64, _dp]),
        "orc_kernel_eval": (_i, [_i, _d, _d, _d, _d, _d, _d, C.POINTER(_d)]),
        "orc_next_smooth": (_i, [_i]),
        "orc_fft2d": (None, [_i, _i, _dp, _i]),
        "orc_cov_create": (_p, [_i, _i, _d, _d, _i, _d, _d, _d, _d, _d]),
        "orc_cov_destroy": (None, [_p]),
        "orc_cov_dims": (None, [_p, C.POINTER(_i), C.POINTER(_i)]),
        "orc_cov_spectrum": (None, [_p, _dp]),
        "orc_cov_apply_count": (C.c_long, [_p]),
        "orc_cov_apply": (_i, [_p, _dp, _ll, _dp]),
        "orc_cov_sample_pair": (_i, [_p, _u64, _u64, _dp, _dp]),
        "orc_trace_ray": (_i, [_i, _i, _d, _d, _d, _d, _d, _d, _i, _llp, _dp]),
        "orc_build_H": (_p, [_i, _i, _d, _d, _i, _dp, _i, _dp]),
        "orc_csr_create": (_p, [_i, _i, _ip, _ip, _dp]),
        "orc_csr_destroy": (None, [_p]),
        "orc_csr_dims": (None, [_p, C.POINTER(_i), C.POINTER(_i), C.POINTER(_ll)]),
        "orc_csr_get": (None, [_p, _ip, _ip, _dp]),
        "orc_ghep": (_p, [_p, _p, _d, _ll, _ll, _u64]),
        "orc_ghep_destroy": (None, [_p]),
        "orc_ghep_rank": (_ll, [_p]),
        "orc_ghep_kept_cols": (_ll, [_p]),
        "orc_ghep_get": (None, [_p, _dp, _p, _p]),
        "orc_fkf_init": (_p, [_p, _p, _d, _ll, _ll, _u64]),
        "orc_fkf_destroy": (None, [_p]),
        "orc_fkf_rank": (_ll, [_p]),
        "orc_fkf_ctx_get": (None, [_p, _p, _p, _p, _p, _p, _p]),
        "orc_fkf_step": (_i, [_p, _dp, _ll]),
        "orc_fkf_state": (None, [_p, C.POINTER(_d), _p, _p, C.POINTER(_i)]),
        "orc_fkf_state_rank": (_ll, [_p]),
        "orc_fkf_set_state": (None, [_p, _d, _dp, _ll, _dp, _i]),
        "orc_variance": (_i, [_p, _dp]),
        "orc_trace_criterion": (_i, [_p, C.POINTER(_d)]),
        "orc_relative_entropy": (_i, [_p, C.POINTER(_d)]),
        "orc_realizations": (_i, [_p, _u64, _i, _dp]),
        "orc_boxcox_map": (_i, [_d, _i, _dp, _ll, _dp]),
        "orc_cov_solve": (_i, [_p, _dp, _d, _dp]),
        "orc_fekf_create": (_p, [_ll, _dp]),
        "orc_fekf_destroy": (None, [_p]),
        "orc_fekf_step": (_i, [_p, _p, _p, _dp, _ll, _d, _d, _ll, _ll, _d, _i, _u64]),
        "orc_fekf_dims": (None, [_p, C.POINTER(_d), C.POINTER(_i), C.POINTER(_ll)]),
        "orc_fekf_read": (None, [_p, _dp, _dp, _dp]),
        "orc_enkf_step": (_i, [_dp, _ll, _ll, _p, _dp, _ll, _p, _d, _u64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class DomainError(ValueError):
    """std::domain_error (boxcox.hpp)."""


def _raise(rc: int):
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 4:
        raise DomainError(msg)  # std::domain_error
    raise RuntimeError(msg)  # std::runtime_error


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ------------------------------------------------------------------ rng.hpp
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def derive_seed(seed: int, tag: int) -> int:
    return int(lib().orc_derive_seed(seed, tag))


def gaussian_vector(n: int, seed: int, stream: int = 0) -> np.ndarray:
    out = np.empty(n)
    lib().orc_gaussian_vector(n, seed, stream, out)
    return out


def gaussian_matrix(rows: int, cols: int, seed: int, base_stream: int = 0) -> np.ndarray:
    """Column-major (Fortran-ordered) rows×cols, column j = stream base+j (rng.hpp:79-86)."""
    out = np.empty(rows * cols)
    lib().orc_gaussian_matrix(rows, cols, seed, base_stream, out)
    return out.reshape(cols, rows).T


def uniforms(n: int, seed: int, stream: int = 0) -> np.ndarray:
    out = np.empty(n)
    lib().orc_uniforms(n, seed, stream, out)
    return out


# ------------------------------------------------------------------ kernel.hpp
POWERED_EXPONENTIAL = 0
MATERN = 1


def kernel_eval(family, theta, length, r, power=1.0, nu=0.5, alpha_scale=0.0) -> float:
    v = _d()
    rc = lib().orc_kernel_eval(family, theta, length, power, nu, alpha_scale, r, C.byref(v))
    if rc:
        _raise(rc)
    return v.value


def next_smooth(n: int) -> int:
    return int(lib().orc_next_smooth(n))


def fft2d(a: np.ndarray, sign: int = -1) -> np.ndarray:
    """Unnormalized 2-D c2c DFT of a complex mx×my array (FFTW convention)."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    buf = a.view(np.float64).ravel().copy()
    lib().orc_fft2d(a.shape[0], a.shape[1], buf, sign)
    return buf.view(np.complex128).reshape(a.shape)


# ------------------------------------------------------------------ covariance.hpp (fft mode)
class CovarianceOperator:
    """covariance.hpp:69-403, FFT mode only (dense mode is desk-scale; tests use numpy)."""

    def __init__(self, nx, ny, lx=1.0, ly=1.0, family=MATERN, theta=1.0, length=0.2, power=1.0,
                 nu=0.5, alpha_scale=0.0):
        self.nx, self.ny = nx, ny
        self.theta = theta
        self._h = lib().orc_cov_create(nx, ny, lx, ly, family, theta, length, power, nu, alpha_scale)
        if not self._h:
            msg = lib().orc_last_error().decode()
            raise (ValueError if "must" in msg or "positive" in msg else RuntimeError)(msg)
        mx, my = _i(), _i()
        lib().orc_cov_dims(self._h, C.byref(mx), C.byref(my))
        self.mx, self.my = mx.value, my.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_cov_destroy(self._h)
            self._h = None

    @property
    def size(self):
        return self.nx * self.ny

    def spectrum(self) -> np.ndarray:
        out = np.empty(self.mx * self.my)
        lib().orc_cov_spectrum(self._h, out)
        return out

    def apply_count(self) -> int:
        return int(lib().orc_cov_apply_count(self._h))

    def apply(self, x: np.ndarray) -> np.ndarray:
        """Γx for a vector or an N×c matrix (column-wise, covariance.hpp:101-115)."""
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        X = x.reshape(-1, 1) if vec else x
        if X.shape[0] != self.size:
            raise ValueError(f"cov_apply: expected vector of length {self.size}, got {X.shape[0]}")
        Xf = np.ascontiguousarray(X.T)
        Y = np.empty_like(Xf)
        rc = lib().orc_cov_apply(self._h, Xf.ravel(), X.shape[1], Y.ravel())
        if rc:
            _raise(rc)
        Y = Y.T
        return Y[:, 0].copy() if vec else np.asfortranarray(Y)

    def sample_pair(self, seed: int, stream: int = 0):
        a = np.empty(self.size)
        b = np.empty(self.size)
        rc = lib().orc_cov_sample_pair(self._h, seed, stream, a, b)
        if rc:
            _raise(rc)
        return a, b


# ------------------------------------------------------------------ tomography.hpp
def trace_ray(nx, ny, src, rec, lx=1.0, ly=1.0):
    cap = 4 * (nx + ny) + 8
    cells = np.empty(cap, dtype=np.int64)
    lens = np.empty(cap)
    n = lib().orc_trace_ray(nx, ny, lx, ly, src[0], src[1], rec[0], rec[1], cap, cells, lens)
    if n < 0:
        _raise(1)
    return cells[:n].copy(), lens[:n].copy()


class Csr:
    """SparseRowMatrix (grid.hpp:15) held by the oracle."""

    def __init__(self, handle):
        self._h = handle
        r, c, nnz = _i(), _i(), _ll()
        lib().orc_csr_dims(handle, C.byref(r), C.byref(c), C.byref(nnz))
        self.rows, self.cols, self.nnz = r.value, c.value, nnz.value

    @classmethod
    def from_arrays(cls, rows, cols, rowptr, col, val):
        return cls(lib().orc_csr_create(rows, cols, np.ascontiguousarray(rowptr, np.int32),
                                        np.ascontiguousarray(col, np.int32),
                                        np.ascontiguousarray(val, np.float64)))

    def arrays(self):
        rowptr = np.empty(self.rows + 1, dtype=np.int32)
        col = np.empty(self.nnz, dtype=np.int32)
        val = np.empty(self.nnz)
        lib().orc_csr_get(self._h, rowptr, col, val)
        return rowptr, col, val

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_csr_destroy(self._h)
            self._h = None


def build_H(nx, ny, sources, receivers, lx=1.0, ly=1.0) -> Csr:
    """tomography.hpp:130-146 (rows source-major; columns ascending)."""
    s = np.ascontiguousarray(np.asarray(sources, dtype=np.float64).reshape(-1, 2)).ravel()
    r = np.ascontiguousarray(np.asarray(receivers, dtype=np.float64).reshape(-1, 2)).ravel()
    h = lib().orc_build_H(nx, ny, lx, ly, len(s) // 2, s, len(r) // 2, r)
    if not h:
        _raise(1)
    return Csr(h)


# ------------------------------------------------------------------ lowrank.hpp / fast_filter.hpp / uq.hpp
def randomized_ghep(cov: CovarianceOperator, h: Csr, sigma2: float, k: int, p: int, seed: int):
    """lowrank.hpp:141-213 with a_apply = HᵀH/σ².  Returns (lambda, U, Ubar, kept_cols)."""
    g = lib().orc_ghep(cov._h, h._h, sigma2, k, p, seed)
    if not g:
        msg = lib().orc_last_error().decode()
        raise (ValueError if "exceeds" in msg or "nonnegative" in msg else RuntimeError)(msg)
    try:
        r = int(lib().orc_ghep_rank(g))
        lam = np.empty(r)
        U = np.empty(cov.size * r)
        Ub = np.empty(cov.size * r)
        lib().orc_ghep_get(g, lam, _ptr(U), _ptr(Ub))
        kept = int(lib().orc_ghep_kept_cols(g))
    finally:
        lib().orc_ghep_destroy(g)
    return lam, U.reshape(r, cov.size).T, Ub.reshape(r, cov.size).T, kept


class FastFilter:
    """fkf_init (fast_filter.hpp:51-75) + a LowRankState advanced by fkf_step (:84-125)."""

    def __init__(self, cov: CovarianceOperator, h: Csr, sigma2, k, p, seed):
        self.cov = cov
        self.h = h
        self.n = cov.size
        self.m = h.rows
        self._f = lib().orc_fkf_init(cov._h, h._h, sigma2, k, p, seed)
        if not self._f:
            msg = lib().orc_last_error().decode()
            raise (ValueError if "must" in msg or "match" in msg or "exceeds" in msg else RuntimeError)(msg)
        self.rank = int(lib().orc_fkf_rank(self._f))

    def __del__(self):
        if getattr(self, "_f", None):
            lib().orc_fkf_destroy(self._f)
            self._f = None

    def context(self, gamma_ht=False):
        r, n, m = self.rank, self.n, self.m
        lam = np.empty(r)
        U = np.empty(n * r)
        Ub = np.empty(n * r)
        G = np.empty(m * m)
        B = np.empty(m * r)
        GH = np.empty(n * m) if gamma_ht else None
        lib().orc_fkf_ctx_get(self._f, _ptr(lam), _ptr(U), _ptr(Ub), _ptr(G), _ptr(B), _ptr(GH))
        out = dict(lam=lam, U=U.reshape(r, n).T, Ubar=Ub.reshape(r, n).T, G=G.reshape(m, m).T,
                   B=B.reshape(r, m).T)
        if gamma_ht:
            out["gamma_ht"] = GH.reshape(m, n).T
        return out

    def step(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        rc = lib().orc_fkf_step(self._f, y, len(y))
        if rc:
            _raise(rc)

    def state(self):
        r = int(lib().orc_fkf_state_rank(self._f))
        a = _d()
        st = _i()
        d = np.empty(r)
        mean = np.empty(self.n)
        lib().orc_fkf_state(self._f, C.byref(a), _ptr(d), _ptr(mean), C.byref(st))
        return dict(alpha=a.value, d=d, mean=mean, step=st.value)

    def set_state(self, alpha, d, mean, step=0):
        d = np.ascontiguousarray(d, dtype=np.float64)
        lib().orc_fkf_set_state(self._f, alpha, d, len(d), np.ascontiguousarray(mean, np.float64), step)

    def variance(self):
        out = np.empty(self.n)
        rc = lib().orc_variance(self._f, out)
        if rc:
            _raise(rc)
        return out

    def trace_criterion(self):
        v = _d()
        rc = lib().orc_trace_criterion(self._f, C.byref(v))
        if rc:
            _raise(rc)
        return v.value

    def relative_entropy(self):
        v = _d()
        rc = lib().orc_relative_entropy(self._f, C.byref(v))
        if rc:
            _raise(rc)
        return v.value

    def realizations(self, seed, count):
        out = np.empty(count * self.n)
        rc = lib().orc_realizations(self._f, seed, count, out)
        if rc:
            _raise(rc)
        return out.reshape(count, self.n).T


# ---------------------------------------------------------------- extended filter
def boxcox(alpha: float, x, which: str) -> np.ndarray:
    """BoxCox::forward / inverse / derivative on a vector (boxcox.hpp:25-75)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    rc = lib().orc_boxcox_map(alpha, {"forward": 0, "inverse": 1, "derivative": 2}[which], x, x.size, out)
    if rc:
        _raise(rc)
    return out


def cov_solve(cov: CovarianceOperator, b, tol: float = 1e-12) -> np.ndarray:
    """CovarianceOperator::solve by CG on the fast matvec (covariance.hpp:118-139)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    rc = lib().orc_cov_solve(cov._h, b, tol, x)
    if rc:
        _raise(rc)
    return x


class ExtendedFilter:
    """LowRankState driven by fekf_step (fast_filter.hpp:127-224) from zero_start with a
    given initial mean (driver.hpp:315-316)."""

    def __init__(self, cov: CovarianceOperator, h: Csr, mean0):
        self.cov, self.h = cov, h
        mean0 = np.ascontiguousarray(mean0, dtype=np.float64)
        self.n = mean0.size
        self._s = lib().orc_fekf_create(self.n, mean0)

    def __del__(self):
        if getattr(self, "_s", None):
            lib().orc_fekf_destroy(self._s)
            self._s = None

    def step(self, y, sigma2, bc_alpha, k_rank=-1, oversampling=20, trunc_tol=1e-5, relinearizations=1, seed=0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        rc = lib().orc_fekf_step(self._s, self.cov._h, self.h._h, y, y.size, sigma2, bc_alpha, k_rank, oversampling,
                                 trunc_tol, relinearizations, seed)
        if rc:
            _raise(rc)

    def state(self):
        a, st, r = _d(), _i(), _ll()
        lib().orc_fekf_dims(self._s, C.byref(a), C.byref(st), C.byref(r))
        mean, d, w = np.empty(self.n), np.empty(r.value), np.empty(self.n * r.value)
        lib().orc_fekf_read(self._s, mean, d, w)
        return {"alpha": a.value, "step": st.value, "mean": mean, "d": d,
                "w": w.reshape(r.value, self.n).T if r.value else np.zeros((self.n, 0))}


# ---------------------------------------------------------------- EnKF (enkf.hpp)
def enkf_step(members, h: Csr, y, cov: CovarianceOperator, sigma2: float, seed: int) -> np.ndarray:
    """enkf_step (enkf.hpp:43-94): returns the new n×ne member matrix."""
    x = np.asfortranarray(np.array(members, dtype=np.float64))
    n, ne = x.shape
    buf = np.ascontiguousarray(x.T).ravel()  # column-major flat
    y = np.ascontiguousarray(y, dtype=np.float64)
    rc = lib().orc_enkf_step(buf, n, ne, h._h, y, y.size, cov._h, sigma2, seed)
    if rc:
        _raise(rc)
    return buf.reshape(ne, n).T.copy()
