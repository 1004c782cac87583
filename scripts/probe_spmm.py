"""SpMM H·X on row-major blocks at a BASELINE config, profiled region (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from tests.helpers import workload_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w, h, ys, s2 = workload_inputs(name)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, 8, 4, w.ghep_seed)
l = k + p
X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(w.N * l))
Z = DeviceArray(w.m * l)
ctx.spmm_rm_device(0, X.ptr, l, Z.ptr); ctx.spmm_device(0, X.ptr, w.N, l, Z.ptr, w.m)
check(lib().fkb_dsync())
check(lib().fkb_profiler(1))
ctx.spmm_rm_device(0, X.ptr, l, Z.ptr)
ctx.spmm_rm_device(1, Z.ptr, l, X.ptr)
ctx.spmm_device(0, X.ptr, w.N, l, Z.ptr, w.m)
check(lib().fkb_dsync())
check(lib().fkb_profiler(0))
print("ok")
