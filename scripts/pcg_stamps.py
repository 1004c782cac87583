"""%globaltimer stamps inside the step's PCG kernel (FKB_PCG_STAMPS=1): start, K staged,
per-iteration, end — averaged over steps 2..n of a BASELINE config (development aid)."""
import os
import sys

os.environ["FKB_PCG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1405_2276_b200 as P  # noqa: E402
from paper_1405_2276_b200 import workloads as W  # noqa: E402
from paper_1405_2276_b200._native import check, lib  # noqa: E402
from tests.helpers import workload_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w, h, ys, s2 = workload_inputs(name, 8)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
rows = []
for i, y in enumerate(ys):
    P.fkf_step(ctx, y)
    st = np.zeros(64, dtype=np.uint64)
    check(lib().fkb_filter_pcg_stamps(ctx._f, st))
    it = ctx.cap_stats()[0]
    if i >= 2 and st[63] > st[0]:
        t = st.astype(np.int64) - int(st[0])
        rows.append((it, t[1], [t[1 + j] for j in range(1, it + 1)], t[63]))
for it, kst, its, end in rows:
    d = np.diff([kst] + its)
    print(f"{name}: iters {it} staged {kst / 1e3:.2f} us, per-iteration {[round(x / 1e3, 2) for x in d]} us, "
          f"end {end / 1e3:.2f} us")
