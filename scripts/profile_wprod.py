"""The offline GHEP's W-block products at a BASELINE config's sizes (default c2: N = 65,536,
l = 320, k = 300) between cudaProfilerStart/Stop, for ncu --profile-from-start off:
the Γ-metric Gram Ȳᵀ(ΓȲ) (k_gram, split-K DMMA) and U = Q·S (k_gemm, DMMA).
Development aid for profiles/ (profiles/round2_ncu_wprod_*.txt)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1405_2276_b200 import workloads as W  # noqa: E402
from paper_1405_2276_b200._native import check, lib  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
k, p = w.ghep_sizes()
l = k + p
L = lib()
Y = torch.randn(l, w.N, dtype=torch.float64, device="cuda")
Z = torch.randn(l, w.N, dtype=torch.float64, device="cuda")
G = torch.empty(l, l, dtype=torch.float64, device="cuda")
S = torch.randn(k, l, dtype=torch.float64, device="cuda")
U = torch.empty(k, w.N, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(2):  # warm-up (workspace allocation, attributes)
    check(L.fkb_dense_product(0, w.N, l, l, ptr(Y), ptr(Z), ptr(G), st))
    check(L.fkb_dense_product(1, w.N, l, k, ptr(Y), ptr(S), ptr(U), st))
torch.cuda.synchronize()
check(L.fkb_profiler(1))
check(L.fkb_dense_product(0, w.N, l, l, ptr(Y), ptr(Z), ptr(G), st))
check(L.fkb_dense_product(1, w.N, l, k, ptr(Y), ptr(S), ptr(U), st))
torch.cuda.synchronize()
check(L.fkb_profiler(0))
print("ok")
