import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray
from tests.helpers import Problem, csr_dense
p = Problem(24, 20, 5, 7, 1, 2e-4)
Hd = csr_dense(p.h); m, n = Hd.shape
fails = 0
for it in range(40):
    cov = P.CovarianceOperator(p.grid, p.spec()); ctx = P.fkf_init(cov, p.h, p.sigma2, 8, 4, 3)
    if it % 2:
        for k in range(3): ctx.step(np.random.default_rng(k).standard_normal(m) * 1e-2)
    for ncols in (256, 300, 320):
        X = np.random.default_rng(ncols).standard_normal((n, ncols))
        dX = DeviceArray.from_host(np.ascontiguousarray(X).ravel())
        dY = DeviceArray.from_host(np.full(m * ncols, np.nan))
        ctx.spmm_rm_device(0, dX.ptr, ncols, dY.ptr)
        G = dY.to_host().reshape(m, ncols); R = Hd @ X
        bad = np.argwhere(~(np.abs(G - R) <= 1e-10 * np.abs(R).max()))
        if len(bad):
            fails += 1
            print(it, ncols, "bad", len(bad), "nan", int(np.isnan(G).sum()), "rows", np.unique(bad[:, 0])[:8], "cols", np.unique(bad[:, 1])[:6], np.unique(bad[:, 1])[-4:])
print("fails", fails)
