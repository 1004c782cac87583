"""PCG iteration counts / verdicts vs conditioning through the test hook (development aid)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1:
    import paper_1405_2276_b200._native as N
    N.LIB_PATH = sys.argv[1]
from paper_1405_2276_b200._native import lib
n = 300
for kappa in (1.5, 3, 10, 30, 100, 1000):
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    K = (Q * np.geomspace(1.0 / kappa, 1.0, n)) @ Q.T
    b = rng.standard_normal(n)
    x, it = np.empty(n), C.c_int()
    rc = lib().fkb_cap_pcg_test(n, np.ascontiguousarray(K.T).ravel(), b, x, C.byref(it), np.zeros(64, dtype=np.uint64))
    ref = np.linalg.solve(K, b)
    print(f"kappa {kappa:7}: rc {rc} iters {it.value:3d} true rel residual {np.linalg.norm(K @ x - b) / np.linalg.norm(b):.2e} "
          f"err {np.linalg.norm(x - ref) / np.linalg.norm(ref):.2e}")
