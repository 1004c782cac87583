"""Runs warm-up steps, then one profiled fkf_step between cudaProfilerStart/Stop
(use with: ncu --profile-from-start off ...).  Development aid for profiles/."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from tests.helpers import workload_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
what = sys.argv[2] if len(sys.argv) > 2 else "step"
w, h, ys, s2 = workload_inputs(name)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
k, p = w.ghep_sizes()
if what == "init":
    check(lib().fkb_profiler(1))
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
if what == "init":
    check(lib().fkb_dsync()); check(lib().fkb_profiler(0)); sys.exit(0)
dys = DeviceArray.from_host(np.stack(ys).ravel())
ctx.steps_async(dys.ptr, 3, w.m); ctx.sync(3)
for mode in (0, 1):
    v = C.c_double(); check(lib().fkb_fp64_peak(mode, C.byref(v))); print(["DFMA", "DMMA"][mode], "peak TFLOP/s", round(v.value, 2))
check(lib().fkb_dsync())
check(lib().fkb_profiler(1))
ctx.steps_async(dys.ptr, 1, w.m)
if w.variance_each_step or w.realizations_per_step:
    X = DeviceArray(w.N * 8); V = DeviceArray(w.N)
    ctx.realizations_device(w.sample_seed, w.realizations_per_step, X.ptr, V.ptr)
check(lib().fkb_dsync())
check(lib().fkb_profiler(0))
ctx.sync(1)
print("ok")
