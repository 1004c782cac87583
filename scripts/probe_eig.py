"""Host Householder-QL vs device block Jacobi on GHEP/add_low_rank-sized symmetric matrices."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
rng = np.random.default_rng(0)
for n in (128, 256, 320, 512, 640, 1024):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.logspace(-8, 6, n) * np.where(rng.random(n) < 0.1, -1, 1)
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    P.sym_eig_device(a)
    t0 = time.perf_counter(); w1, z1 = P.sym_eig(a); t1 = time.perf_counter()
    w2, z2, sw = P.sym_eig_device(a); t2 = time.perf_counter()
    ref = np.sort(lam)
    print(f"n={n}: host {1e3*(t1-t0):.1f} ms err {np.max(np.abs(w1-ref))/np.abs(ref).max():.1e} | "
          f"device {1e3*(t2-t1):.1f} ms sweeps {sw} err {np.max(np.abs(w2-ref))/np.abs(ref).max():.1e} "
          f"res {np.linalg.norm(a@z2 - z2*w2)/np.linalg.norm(a):.1e} orth {np.abs(z2.T@z2-np.eye(n)).max():.1e}", flush=True)
