"""Per-iteration timing of the capacitance PCG kernel (development aid)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1405_2276_b200._native import lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(0)
F = rng.standard_normal((n, n)) / np.sqrt(n)
K = np.eye(n) - 0.05 * F.T @ F / 2 + np.diag(rng.uniform(0, 0.1, n))
b = rng.standard_normal(n)
Kc = np.ascontiguousarray(K.T).ravel()
x = np.empty(n); st = np.zeros(64, dtype=np.uint64); it = C.c_int()
for rep in range(3):
    rc = lib().fkb_cap_pcg_test(n, Kc, b, x, C.byref(it), st)
ref = np.linalg.solve(K, b)
print("rc", rc, "iters", it.value, "cond", np.linalg.cond(K), "rel err", np.linalg.norm(x - ref) / np.linalg.norm(ref))
t0 = int(st[0])
print("stage", int(st[1]) - t0, "ns")
for k in range(1, min(it.value, 60)):
    print(f" iter {k}: {int(st[1 + k]) - int(st[k])} ns")
print("total", int(st[63]) - t0, "ns")
if it.value > 4:
    b = int(st[39])
    print("iter 3 (SM cycles): sent", int(st[40]) - b, "| waited", int(st[41]) - b, "| shuffled", int(st[45]) - b,
          "| decided", int(st[46]) - b, "| flag", int(st[42]) - b, "| matvec", int(st[43]) - b, "| update", int(st[44]) - b)
