"""PCG kernel phase stamps inside a real c2 filter step (run with FKB_PCG_STAMPS=1)."""
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
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
dys = DeviceArray.from_host(np.stack(ys).ravel())
ctx.steps_async(dys.ptr, 4, w.m); ctx.sync(4)
st = np.zeros(64, dtype=np.uint64)
check(lib().fkb_filter_pcg_stamps(ctx._f, st))
t0 = int(st[0]); it = ctx.cap_stats()[0]
print("iters", it)
print("K staging + initial exchange + matvec:", int(st[1]) - t0, "ns")
for q in range(1, it + 1):
    if st[1 + q]:
        print(f" iter {q}: {int(st[1 + q]) - int(st[q])} ns")
print("final check + exit:", int(st[63]) - int(st[1 + it]), "ns")
print("total", int(st[63]) - t0, "ns")
if st[39]:
    b = int(st[39])
    print("iter 3 phases (SM cycles from start): send", int(st[40]) - b, "| wait", int(st[41]) - b,
          "| shuffled", int(st[45]) - b, "| decided", int(st[46]) - b, "| flag", int(st[42]) - b, "| matvec", int(st[43]) - b, "| update", int(st[44]) - b)
