"""Quick timing probe of the hot path at a BASELINE config (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from tests.helpers import workload_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w, h, ys, s2 = workload_inputs(name)
kern = P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu)
t0 = time.perf_counter()
cov = P.CovarianceOperator(P.Grid(w.n, w.n), kern)
t1 = time.perf_counter()
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
check(lib().fkb_dsync())
t2 = time.perf_counter()
print(f"{name}: cov {t1-t0:.3f}s fkf_init {t2-t1:.3f}s rank {ctx.rank()} kept {ctx.kept_cols}", flush=True)
dys = DeviceArray.from_host(np.stack(ys).ravel())
ctx.steps_async(dys.ptr, 2, w.m); ctx.sync(2)
check(lib().fkb_dsync())
t = time.perf_counter()
ctx.steps_async(C_ptr := dys.ptr, nsteps, 0) if False else None
for i in range(nsteps):
    ctx.steps_async(dys.ptr, 1, w.m)
ctx.sync(nsteps)
t3 = time.perf_counter()
print(f"steps: {(t3-t)/nsteps*1e3:.3f} ms/step ({nsteps} steps, launches/step {ctx.launches_per_step()}) "
      f"cap PCG (iters, fallback) {ctx.cap_stats()}", flush=True)
# Γ·X on m+l columns
N = w.N; c = w.m + k + p
X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(N * c))
Y = DeviceArray(N * c)
cov.apply_device(X.ptr, N, c, Y.ptr, N); check(lib().fkb_dsync())
t = time.perf_counter(); reps = 3
for _ in range(reps): cov.apply_device(X.ptr, N, c, Y.ptr, N)
check(lib().fkb_dsync()); t4 = time.perf_counter()
dt = (t4 - t) / reps
my, mx, nx = cov.my, cov.mx, w.n
F = 5 * nx * my * np.log2(my) + 10 * (my // 2 + 1) * mx * np.log2(mx) + 2 * mx * (my // 2 + 1)
print(f"GammaX: {c} cols {dt*1e3:.2f} ms -> {F*c/dt/1e12:.2f} TFLOP/s (pruned R2C convention)", flush=True)
# SpMM H·X with l columns
l = k + p
Z = DeviceArray(w.m * l)
ctx.spmm_device(0, X.ptr, N, l, Z.ptr, w.m); check(lib().fkb_dsync())
t = time.perf_counter()
for _ in range(reps): ctx.spmm_device(0, X.ptr, N, l, Z.ptr, w.m)
check(lib().fkb_dsync()); dt = (time.perf_counter() - t) / reps
B = 12 * h.nnz + 4 * (h.rows + 1) + 8 * (N + w.m) * l
print(f"SpMM H·X (l={l}): {dt*1e6:.1f} us -> {B/dt/1e9:.0f} GB/s", flush=True)
ctx.spmm_rm_device(0, X.ptr, l, Z.ptr); check(lib().fkb_dsync())
t = time.perf_counter()
for _ in range(reps): ctx.spmm_rm_device(0, X.ptr, l, Z.ptr)
check(lib().fkb_dsync()); dt = (time.perf_counter() - t) / reps
print(f"SpMM H·X row-major (l={l}): {dt*1e6:.1f} us -> {B/dt/1e9:.0f} GB/s", flush=True)
ctx.spmm_rm_device(1, Z.ptr, l, X.ptr); check(lib().fkb_dsync())
t = time.perf_counter()
for _ in range(reps): ctx.spmm_rm_device(1, Z.ptr, l, X.ptr)
check(lib().fkb_dsync()); dt = (time.perf_counter() - t) / reps
print(f"SpMM Hᵀ·Y row-major (l={l}): {dt*1e6:.1f} us -> {B/dt/1e9:.0f} GB/s", flush=True)
ctx.spmm_device(1, Z.ptr, w.m, l, X.ptr, N); check(lib().fkb_dsync())
t = time.perf_counter()
for _ in range(reps): ctx.spmm_device(1, Z.ptr, w.m, l, X.ptr, N)
check(lib().fkb_dsync()); dt = (time.perf_counter() - t) / reps
print(f"SpMM Hᵀ·Y (l={l}): {dt*1e6:.1f} us -> {B/dt/1e9:.0f} GB/s", flush=True)
ctx.reset()
print("phases (ms):", {k: round(v, 4) for k, v in ctx.phase_times(5).items()}, flush=True)
