"""One profiling entry point for profiles/ (development aid, not product code).

    python scripts/profile.py MODE [CONFIG] [ARG]

Each mode runs its warm-up outside, then the region of interest between
cudaProfilerStart/Stop, so `ncu --profile-from-start off …` captures exactly that region:

  step   one fkf_step after 3 warm steps (the fused step + diag Σ + realizations when the
         config draws them, as bench.py runs it)
  init   fkf_init (spectrum, GHEP, G = HΓHᵀ and its eigendecomposition)
  wprod  the GHEP's W-block products at the config's sizes: the Γ-metric Gram Ȳᵀ(ΓȲ)
         (k_gram), U = Q·S (k_gemm) and the symmetric capacitance Gram (k_gram_sym)
  gx     the batched Γ·X on ARG columns (default 256)
  spmm   H·X and Hᵀ·Y on row-major blocks of l = k + p columns, then column-major H·X
  enkf   ARG (default 4) EnKF steps with NE members (env, default 1000), timed
  fekf   ARG (default 3) extended-filter steps at the config's grid, timed with phase info
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1405_2276_b200 as P  # noqa: E402
from paper_1405_2276_b200 import workloads as W  # noqa: E402
from paper_1405_2276_b200._native import DeviceArray, check, lib  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "step"
name = sys.argv[2] if len(sys.argv) > 2 else "c2"
arg = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = W.CONFIGS[name]
cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
k, p = w.ghep_sizes()
L = lib()


def region(fn):
    check(L.fkb_dsync())
    check(L.fkb_profiler(1))
    fn()
    check(L.fkb_dsync())
    check(L.fkb_profiler(0))


if mode in ("step", "init", "spmm"):
    from tests.helpers import workload_inputs
    w, h, ys, s2 = workload_inputs(name)
    if mode == "init":
        region(lambda: P.fkf_init(cov, h, s2, k, p, w.ghep_seed))
    elif mode == "step":
        ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
        dys = DeviceArray.from_host(np.stack(ys).ravel())
        ctx.steps_async(dys.ptr, 3, w.m)
        ctx.sync(3)

        uq = bool(w.variance_each_step or w.realizations_per_step)
        X, V = DeviceArray(w.N * 8), DeviceArray(w.N)
        cnt = int(w.realizations_per_step or 0)

        def one():  # the step as bench.py runs it: fused step + UQ when the config draws UQ
            if uq:
                ctx.step_uq_device(dys.ptr, w.sample_seed, cnt, X.ptr, V.ptr)
            else:
                ctx.steps_async(dys.ptr, 1, w.m)
        if uq:
            for _ in range(3):
                one()
        region(one)
        ctx.sync(1)
    else:
        ctx = P.fkf_init(cov, h, s2, 8, 4, w.ghep_seed)
        l = k + p
        X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(w.N * l))
        Z = DeviceArray(w.m * l)
        ctx.spmm_rm_device(0, X.ptr, l, Z.ptr)
        ctx.spmm_device(0, X.ptr, w.N, l, Z.ptr, w.m)

        def spmm():
            ctx.spmm_rm_device(0, X.ptr, l, Z.ptr)
            ctx.spmm_rm_device(1, Z.ptr, l, X.ptr)
            ctx.spmm_device(0, X.ptr, w.N, l, Z.ptr, w.m)
        region(spmm)
elif mode == "wprod":
    import torch
    l = k + p
    Y = torch.randn(l, w.N, dtype=torch.float64, device="cuda")
    Z = torch.randn(l, w.N, dtype=torch.float64, device="cuda")
    G = torch.empty(l, l, dtype=torch.float64, device="cuda")
    S = torch.randn(k, l, dtype=torch.float64, device="cuda")
    U = torch.empty(k, w.N, dtype=torch.float64, device="cuda")
    E = torch.randn(k, w.m, dtype=torch.float64, device="cuda")
    K = torch.empty(k, k, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def wprod():
        check(L.fkb_dense_product(0, w.N, l, l, ptr(Y), ptr(Z), ptr(G), st))
        check(L.fkb_dense_product(1, w.N, l, k, ptr(Y), ptr(S), ptr(U), st))
        check(L.fkb_dense_product(2, w.m, k, k, ptr(E), ptr(E), ptr(K), st))
    for _ in range(2):  # workspace allocation, attributes
        wprod()
    torch.cuda.synchronize()
    region(wprod)
elif mode == "gx":
    ncols = arg or 256
    X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(w.N * ncols))
    Y = DeviceArray(w.N * ncols)
    cov.apply_device(X.ptr, w.N, ncols, Y.ptr, w.N)
    region(lambda: cov.apply_device(X.ptr, w.N, ncols, Y.ptr, w.N))
elif mode == "enkf":
    ne = int(os.environ.get("NE", "1000"))
    w, h, ys, s2 = W.problem(name, arg or 4)
    ens = P.Ensemble(cov, h, ne)
    for i, y in enumerate(ys):
        t0 = time.perf_counter()
        ens.step(y, s2, W.derive_seed(1011, i + 1))
        print(f"{name} N_e={ne} step {i + 1}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
elif mode == "fekf":
    w, h, ys, s2 = W.problem(name, arg or 3)
    g = P.ExtendedFilter(cov, h, np.full(w.N, -1.0))
    for i, y in enumerate(ys):
        t0 = time.perf_counter()
        g.step(y, s2, P.BoxCox(1.0), P.FekfOptions(k_rank=k, oversampling=p, trunc_tol=1e-5, seed=i))
        print(f"{name} fekf step {i + 1}: {1e3 * (time.perf_counter() - t0):.1f} ms rank {g.rank()}",
              g.last_step_info(), flush=True)
else:
    sys.exit(f"unknown mode {mode}")
print("ok")
