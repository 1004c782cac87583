"""Phase timing of the cluster capacitance factor+solve kernel (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1405_2276_b200._native import lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(0)
F = rng.standard_normal((n, n)) / np.sqrt(3 * n)
K = np.eye(n) - F.T @ F * 0.5
b = rng.standard_normal(n)
Kc = np.ascontiguousarray(K.T).ravel()
L = np.empty(n * n); x = np.empty(n); st = np.zeros(160, dtype=np.uint64)
for rep in range(3):
    rc = lib().fkb_chol_solve_small(n, Kc, b, L, x, st)
print("rc", rc, "rel err", np.linalg.norm(x - np.linalg.solve(K, b)) / np.linalg.norm(np.linalg.solve(K, b)))
T = (n + 31) // 32
t0 = int(st[0])
for j in range(T):
    s = [int(st[6 * j + q]) for q in range(6)]
    print(f"panel {j}: A {s[1]-s[0]} | barA {s[2]-s[1]} | B {s[3]-s[2]} | barB {s[4]-s[3]} | C+bar {s[5]-s[4]} ns")
prev = int(st[120]); print("backward start", prev - t0)
for j in range(T):
    v = int(st[121 + j]); print(f" back {j}: {v - prev} ns"); prev = v
print("total", prev - t0, "ns")
cyc = int(st[159]) - int(st[158])
print("SM clock during kernel: %.0f MHz" % (cyc / (prev - t0) * 1e3))
print("initial diag factor (A0):", int(st[151]) - int(st[150]), "ns")
