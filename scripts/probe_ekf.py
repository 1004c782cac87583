"""Extended filter: per-step parity errors against the oracle on the reference's fekf test
problems, and a timed run at a BASELINE-size grid (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import EXPERIMENT, Problem, low_rank_cov, rel_err

cases = {
    "identity": (Problem(10, 10, 2, 4, 8, 2e-4), 1.0, 0.0, 1, 900, -1.0),
    "boxcox2": (Problem(8, 8, 2, 4, 5, 2e-4, kernel=dict(EXPERIMENT, theta=1e-4)), 2.0, 0.0, 1, 901, None),
    "relin3": (Problem(8, 8, 2, 4, 3, 2e-4), 4.0, 0.0, 3, 902, None),
    "trunc": (Problem(12, 12, 3, 8, 6, 2e-4, kernel=dict(EXPERIMENT, theta=1e-5, power=1.0)), 2.0, 1e-5, 1, 903, None),
    "mid24": (Problem(24, 24, 6, 8, 3, 1e-4, kernel=dict(EXPERIMENT, theta=1e-4)), 3.0, 0.0, 3, 904, None),
}
for name, (p, bc, tol, relin, tag, m0) in cases.items():
    n = p.nx * p.ny
    mean0 = np.full(n, m0 if m0 is not None else O.boxcox(bc, [1e-4], "forward")[0])
    cov = P.CovarianceOperator(p.grid, p.spec())
    g = P.ExtendedFilter(cov, p.h, mean0)
    o = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), mean0)
    gam = p.gamma()
    worst = [0.0, 0.0, 0.0]
    for k, y in enumerate(p.obs):
        seed = W.derive_seed(tag, k)
        g.step(y, p.sigma2, P.BoxCox(bc), P.FekfOptions(k_rank=p.h.rows, trunc_tol=tol, relinearizations=relin, seed=seed))
        o.step(y, p.sigma2, bc, k_rank=p.h.rows, trunc_tol=tol, relinearizations=relin, seed=seed)
        gs, os_ = g.state(), o.state()
        em = rel_err(gs["mean"], os_["mean"])
        ec = rel_err(low_rank_cov(gs["alpha"], gs["w"], gs["d"], gam), low_rank_cov(os_["alpha"], os_["w"], os_["d"], gam))
        kk = min(len(gs["d"]), len(os_["d"]))
        ed = float(np.max(np.abs(gs["d"][:kk] - os_["d"][:kk])) / gs["alpha"]) if kk else 0.0
        worst = [max(worst[0], em), max(worst[1], ec), max(worst[2], ed)]
        print(f"{name} step {k+1}: rank gpu {len(gs['d'])} oracle {len(os_['d'])} mean {em:.2e} cov {ec:.2e} d {ed:.2e}")
    print(f"{name} WORST mean {worst[0]:.2e} cov {worst[1]:.2e} d {worst[2]:.2e}", flush=True)

# timing at BASELINE grids: c0 (64², m = 256) and c2 (256², m = 2048), Box–Cox 2, rank cap as BASELINE
for cfg in sys.argv[1:]:
    w, h, ys, s2 = W.problem(cfg, 4)
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
    k, pp = w.ghep_sizes()
    mean0 = np.full(w.N, -1.0)
    g = P.ExtendedFilter(cov, h, mean0)
    ts = []
    for i, y in enumerate(ys[:4]):
        t0 = time.perf_counter()
        g.step(y, s2, P.BoxCox(1.0), P.FekfOptions(k_rank=k, oversampling=pp, trunc_tol=1e-5, seed=i))
        ts.append(time.perf_counter() - t0)
        print(cfg, "step", i + 1, f"{ts[-1]*1e3:.1f} ms rank {g.rank()}", g.last_step_info(), flush=True)
