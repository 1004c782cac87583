"""Per-step UQ cost (diag Σ + count realizations in one U pass) at a config (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from tests.helpers import workload_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w, h, ys, s2 = workload_inputs(name)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
dys = DeviceArray.from_host(np.stack(ys).ravel())
ctx.steps_async(dys.ptr, 3, w.m); ctx.sync(3)
X = DeviceArray(w.N * count); V = DeviceArray(w.N)
ctx.realizations_device(w.sample_seed, count, X.ptr, V.ptr)  # draws + Ūᵀz cached here
check(lib().fkb_dsync())
reps = 20
t = time.perf_counter()
for _ in range(reps):
    ctx.realizations_device(w.sample_seed, count, X.ptr, V.ptr)
check(lib().fkb_dsync())
dt = (time.perf_counter() - t) / reps
print(f"{name}: UQ (var + {count} realizations) {dt*1e6:.1f} us; U {w.N*k*8/1e6:.0f} MB -> {w.N*k*8/dt/1e9:.0f} GB/s")
t = time.perf_counter()
for i in range(reps):
    ctx.steps_async(dys.ptr, 1, w.m)
    ctx.realizations_device(w.sample_seed, count, X.ptr, V.ptr)
ctx.sync(reps)
dt = (time.perf_counter() - t) / reps
print(f"{name}: step + UQ {dt*1e3:.3f} ms -> {1/dt:.0f} steps/s")
