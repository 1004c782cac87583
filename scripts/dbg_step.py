import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1405_2276_b200 as P
from tests.helpers import Problem
p = Problem(12, 12, 3, 8, 3, 2e-4)
ctx = P.fkf_init(P.CovarianceOperator(p.grid, p.spec()), p.h, p.sigma2, 16, 20, 11)
from paper_1405_2276_b200._native import DeviceArray
d = DeviceArray.from_host(p.obs[0])
from paper_1405_2276_b200._native import lib, check
import ctypes as C
check(lib().fkb_h2d(C.c_void_p(0), C.c_void_p(0), 0))
try:
    print(ctx.phase_times(1))
except Exception as e:
    print("ERR", e)
