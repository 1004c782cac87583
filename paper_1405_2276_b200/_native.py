"""ctypes loader for libfastkf_b200.so (the sm_100a product library).

There is no fallback: if the shared library is missing the import fails loudly, and every
compute entry point runs CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfastkf_b200.so")

_d = C.c_double
_i = C.c_int
_ll = C.c_longlong
_u64 = C.c_uint64
_p = C.c_void_p
_sz = C.c_size_t
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_llp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_PI = C.POINTER(_i)
_PD = C.POINTER(_d)
_PLL = C.POINTER(_ll)

# name -> (restype, argtypes); must match include/fastkf_b200.h
SIGNATURES = {
    "fkb_last_error": (C.c_char_p, []),
    "fkb_launch_count": (C.c_ulonglong, []),
    "fkb_version": (_i, []),
    "fkb_device_count": (_i, []),
    "fkb_kernel_eval": (_i, [_i, _d, _d, _d, _d, _d, _d, _PD]),
    "fkb_next_smooth": (_i, [_i]),
    "fkb_trace_ray": (_i, [_i, _i, _d, _d, _d, _d, _d, _d, _i, _llp, _dp, _PI]),
    "fkb_build_H": (_i, [_i, _i, _d, _d, _i, _dp, _i, _dp, _PI, _PLL, _p, _p, _p, _ll]),
    "fkb_sym_eig": (_i, [_i, _dp, _dp, _dp]),
    "fkb_cov_create": (_i, [_i, _i, _d, _d, _i, _d, _d, _d, _d, _d, C.POINTER(_p)]),
    "fkb_cov_destroy": (None, [_p]),
    "fkb_cov_dims": (_i, [_p, _PI, _PI]),
    "fkb_cov_spectrum": (_i, [_p, _dp]),
    "fkb_cov_apply": (_i, [_p, _p, _ll, _i, _p, _ll]),
    "fkb_cov_apply_device": (_i, [_p, _p, _ll, _i, _p, _ll]),
    "fkb_cov_sample_pair": (_i, [_p, _u64, _u64, _dp, _dp]),
    "fkb_cov_apply_count": (_ll, [_p]),
    "fkb_cov_stream": (_p, [_p]),
    "fkb_gaussian_matrix": (_i, [_ll, _i, _u64, _u64, _dp]),
    "fkb_fkf_init": (_i, [_p, _i, _i, _ip, _ip, _dp, _d, _ll, _ll, _u64, C.POINTER(_p)]),
    "fkb_sym_eig_device": (_i, [_i, _dp, _dp, _dp, C.POINTER(_i)]),
    "fkb_sym_eig_tridiag": (_i, [_i, _dp, _dp, _dp]),
    "fkb_enkf_init": (_i, [_p, _i, _i, _ip, _ip, _dp, _i, C.POINTER(_p)]),
    "fkb_enkf_destroy": (None, [_p]),
    "fkb_enkf_step": (_i, [_p, _dp, _ll, _d, _u64]),
    "fkb_enkf_members": (_i, [_p, _dp]),
    "fkb_enkf_set_members": (_i, [_p, _dp]),
    "fkb_enkf_mean": (_i, [_p, _dp]),
    "fkb_fkf_step_uq": (_i, [_p, _p, _ll, _u64, _i, _p, _p, _p, _p, _p]),
    "fkb_fkf_step_uq_device": (_i, [_p, _p, _u64, _i, _p, _p]),
    "fkb_filter_ghep_residual": (_i, [_p, _dp]),
    "fkb_ekf_create": (_i, [_p, _i, _i, _ip, _ip, _dp, C.POINTER(_p)]),
    "fkb_ekf_destroy": (None, [_p]),
    "fkb_ekf_reset": (_i, [_p, _dp]),
    "fkb_ekf_step": (_i, [_p, _dp, _ll, _d, _d, _ll, _ll, _d, _i, _u64]),
    "fkb_ekf_state": (_i, [_p, C.POINTER(_d), C.POINTER(_i), C.POINTER(_i)]),
    "fkb_ekf_read": (_i, [_p, _p, _p, _p, _p]),
    "fkb_ekf_last": (_i, [_p, C.POINTER(_i), C.POINTER(_i)]),
    "fkb_ekf_uq": (_i, [_p, C.POINTER(_d), C.POINTER(_d)]),
    "fkb_filter_destroy": (None, [_p]),
    "fkb_filter_rank": (_i, [_p, _PI, _PI]),
    "fkb_filter_lambda": (_i, [_p, _dp]),
    "fkb_filter_get": (_i, [_p, _i, _dp]),
    "fkb_fkf_step": (_i, [_p, _p, _ll]),
    "fkb_fkf_step_state": (_i, [_p, _p, _ll, _p, _p, _p]),
    "fkb_fkf_run": (_i, [_p, _p, _i, _ll, _p, _p, _ll, _p, _ll]),
    "fkb_fkf_run_uq": (_i, [_p, _p, _i, _ll, C.c_uint64, _i, _p, _p, _p, _p, _ll, _p, _ll]),
    "fkb_fkf_step_device": (_i, [_p, _p]),
    "fkb_fkf_steps_async": (_i, [_p, _p, _i, _ll]),
    "fkb_fkf_sync": (_i, [_p, _i]),
    "fkb_filter_state": (_i, [_p, _PD, _PI, _PI, _p, _p]),
    "fkb_filter_set_state": (_i, [_p, _d, _i, _i, _p, _p]),
    "fkb_filter_reset": (_i, [_p]),
    "fkb_filter_mean_device": (_i, [_p, C.POINTER(_p)]),
    "fkb_variance": (_i, [_p, _dp]),
    "fkb_variance_device": (_i, [_p, _p]),
    "fkb_trace_criterion": (_i, [_p, _PD]),
    "fkb_relative_entropy": (_i, [_p, _PD]),
    "fkb_realizations": (_i, [_p, _u64, _i, _dp]),
    "fkb_realizations_device": (_i, [_p, _u64, _i, _p, _p]),
    "fkb_realizations_with_variance": (_i, [_p, _u64, _i, _p, _p]),
    "fkb_filter_spmm": (_i, [_p, _i, _p, _ll, _i, _p, _ll]),
    "fkb_filter_stream": (_p, [_p]),
    "fkb_filter_spmm_rm": (_i, [_p, _i, _p, _i, _p]),
    "fkb_filter_launches_per_step": (_i, [_p]),
    "fkb_filter_set_solver": (_i, [_p, _i]),
    "fkb_filter_eig_sweeps": (_i, [_p]),
    "fkb_filter_cap_stats": (_i, [_p, _PI, _PI]),
    "fkb_filter_set_pcg_maxit": (_i, [_p, _i]),
    "fkb_filter_pcg_stamps": (_i, [_p, np.ctypeslib.ndpointer(dtype=np.uint64)]),
    "fkb_filter_get_eig": (_i, [_p, _p, _p]),
    "fkb_filter_phase_times": (_i, [_p, _i, _dp, C.c_char_p, _i, _PI]),
    "fkb_filter_graph_timing": (_i, [_p, _i]),
    "fkb_filter_graph_phase_times": (_i, [_p, _dp, C.c_char_p, _i, _PI]),
    "fkb_fp64_peak": (_i, [_i, _PD]),
    "fkb_l2_peak": (_i, [_i, _PD]),
    "fkb_chol_solve_small": (_i, [_i, _dp, _dp, _dp, _dp, np.ctypeslib.ndpointer(dtype=np.uint64)]),
    "fkb_cap_pcg_test": (_i, [_i, _dp, _dp, _dp, _PI, np.ctypeslib.ndpointer(dtype=np.uint64)]),
    "fkb_set_device": (_i, [_i]),
    "fkb_profiler": (_i, [_i]),
    "fkb_dmalloc": (_i, [C.POINTER(_p), _sz]),
    "fkb_dfree": (_i, [_p]),
    "fkb_h2d": (_i, [_p, _p, _sz]),
    "fkb_d2h": (_i, [_p, _p, _sz]),
    "fkb_dsync": (_i, []),
    "fkb_realization_at": (_i, [_p, _u64, _u64, _dp]),
    "fkb_lowrank_uq": (_i, [_p, _ll, _i, _d, _p, _p, _ll, _p, _p]),
    "fkb_ekf_realizations": (_i, [_p, _u64, _u64, _i, _p, _p]),
    "fkb_dense_product": (_i, [_i, _ll, _i, _i, _p, _p, _p, _p]),
    "fkb_ghep_run": (_i, [_p, _i, _i, _ip, _ip, _dp, _d, _ll, _ll, _u64, C.POINTER(_p)]),
    "fkb_ghep_destroy": (None, [_p]),
    "fkb_ghep_info": (_i, [_p, _PI, _PI]),
    "fkb_ghep_get": (_i, [_p, _i, _dp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1405_2276_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class CudaError(RuntimeError):
    pass


class DomainError(ValueError):
    """std::domain_error (the Box–Cox maps, boxcox.hpp:58-75)."""


def check(rc: int):
    if rc == 0:
        return
    msg = lib().fkb_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise CudaError(msg)
    if rc == 4:
        raise DomainError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class DeviceArray:
    """Minimal owning device buffer of float64 (plumbing for benches/tests without torch)."""

    def __init__(self, n: int):
        self.n = int(n)
        self.ptr = C.c_void_p()
        check(lib().fkb_dmalloc(C.byref(self.ptr), max(self.n, 1) * 8))

    @classmethod
    def from_host(cls, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        d = cls(a.size)
        if a.size:
            check(lib().fkb_h2d(d.ptr, ptr(a), a.size * 8))
        return d

    def to_host(self) -> np.ndarray:
        out = np.empty(self.n)
        if self.n:
            check(lib().fkb_d2h(ptr(out), self.ptr, self.n * 8))
        return out

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value and _lib is not None:
            _lib.fkb_dfree(self.ptr)
            self.ptr = None
