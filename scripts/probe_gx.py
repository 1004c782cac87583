"""Device time of the batched Γ·X on the offline block (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from paper_1405_2276_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
ncols = int(sys.argv[2]) if len(sys.argv) > 2 else 256
w = W.CONFIGS[name]
cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(w.N * ncols))
Y = DeviceArray(w.N * ncols)
cov.apply_device(X.ptr, w.N, ncols, Y.ptr, w.N)
check(lib().fkb_dsync())
check(lib().fkb_profiler(1))
cov.apply_device(X.ptr, w.N, ncols, Y.ptr, w.N)
check(lib().fkb_dsync())
check(lib().fkb_profiler(0))
print("ok")
