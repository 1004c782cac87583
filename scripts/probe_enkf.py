"""EnKF step timing at BASELINE grids (N_e members), GPU vs the oracle on the host (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W

ne = int(os.environ.get("NE", "1000"))
for cfg in sys.argv[1:]:
    w, h, ys, s2 = W.problem(cfg, 4)
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
    ens = P.Ensemble(cov, h, ne)
    ts = []
    for k, y in enumerate(ys[:4]):
        t0 = time.perf_counter()
        ens.step(y, s2, W.derive_seed(1011, k + 1))
        ts.append(time.perf_counter() - t0)
    print(f"{cfg} N_e={ne}: GPU step ms {[round(1e3 * t, 2) for t in ts]}", flush=True)
    if os.environ.get("CPU") and cfg in ("c0",):
        oc = O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu)
        oh = O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val)
        x = np.zeros((w.N, ne))
        t0 = time.perf_counter()
        x = O.enkf_step(x, oh, ys[0], oc, s2, W.derive_seed(1011, 1))
        print(f"{cfg} N_e={ne}: oracle step {time.perf_counter() - t0:.2f} s ({O.max_threads()} threads)", flush=True)
