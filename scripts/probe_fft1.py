"""Device time of one single-vector Γ·x (development aid)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cov = P.CovarianceOperator(P.Grid(n, n), P.KernelSpec(family=1, theta=1.0, length=0.1, nu=0.5))
X = DeviceArray.from_host(np.random.default_rng(0).standard_normal(n * n))
Y = DeviceArray(n * n)
for _ in range(5): cov.apply_device(X.ptr, n * n, 1, Y.ptr, n * n)
check(lib().fkb_dsync())
import time
reps = 200
t = time.perf_counter()
for _ in range(reps): cov.apply_device(X.ptr, n * n, 1, Y.ptr, n * n)
check(lib().fkb_dsync())
print(f"n={n} torus {cov.mx}x{cov.my}: {(time.perf_counter() - t) / reps * 1e6:.1f} us per apply (back-to-back, launch-bound floor incl.)")
