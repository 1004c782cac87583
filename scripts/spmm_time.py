"""Times the offline SpMM H·X (and Hᵀ·Y) on row-major blocks at a BASELINE config with CUDA
events (development aid for the FKB_SPMM_QU sweep; bench.py reports the default shape)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1405_2276_b200 as P  # noqa: E402
from paper_1405_2276_b200 import workloads as W  # noqa: E402
from paper_1405_2276_b200._native import check, lib  # noqa: E402
from tests.helpers import workload_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w, h, ys, s2 = workload_inputs(name)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, 8, 4, w.ghep_seed)
l = k + p
X = torch.randn(w.N, l, dtype=torch.float64, device="cuda")
Z = torch.empty(w.m, l, dtype=torch.float64, device="cuda")
ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(ctx.stream)  # the library's stream
out = {}
for which, src, dst in ((0, X, Z), (1, Z, X)):
    ctx.spmm_rm_device(which, ptr(src), l, ptr(dst))
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(10):
        ctx.spmm_rm_device(which, ptr(src), l, ptr(dst))
    b.record(st)
    torch.cuda.synchronize()
    out[which] = a.elapsed_time(b) / 10
# correctness of the timed kernel: H·X against scipy on the host
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
Hs = sp.csr_matrix((np.asarray(h.val), np.asarray(h.col), np.asarray(h.rowptr)), shape=(w.m, w.N))
ctx.spmm_rm_device(0, ptr(X), l, ptr(Z))
torch.cuda.synchronize()
ref = Hs @ X.cpu().numpy()
err = np.abs(Z.cpu().numpy() - ref).max() / np.abs(ref).max()
pk = C.c_double()
check(lib().fkb_l2_peak(32, C.byref(pk)))
alg = 12 * h.nnz + 4 * (h.rows + 1) + 8 * (w.N + w.m) * l
print(f"{name} QU={os.environ.get('FKB_SPMM_QU', 'default')}: H·X {out[0] * 1e3:.1f} us = {alg / out[0] / 1e6:.0f} GB/s alg, "
      f"L2 {8 * h.nnz * l / out[0] / 1e6:.0f} GB/s of {pk.value:.0f} ({8 * h.nnz * l / out[0] / 1e6 / pk.value:.2f}); "
      f"Hᵀ·Y {out[1] * 1e3:.1f} us; max rel err vs scipy {err:.1e}", flush=True)
