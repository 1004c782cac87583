"""Host Householder-QL vs the GPU tridiagonal path (tdeig.cu) vs the device block Jacobi on
GHEP/add_low_rank-sized symmetric matrices: time, eigenvalue error, residual, orthogonality."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_2276_b200 as P
from paper_1405_2276_b200 import fastkf as F
rng = np.random.default_rng(0)
for n in (128, 320, 512, 640, 1024):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.logspace(-8, 6, n) * np.where(rng.random(n) < 0.1, -1, 1)
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    F.sym_eig_tridiag(a)
    ref = np.sort(lam)
    for name, fn in (("host", F.sym_eig), ("tridiag", F.sym_eig_tridiag)):
        t0 = time.perf_counter(); w, z = fn(a)[:2]; t1 = time.perf_counter()
        print(f"n={n} {name}: {1e3*(t1-t0):.1f} ms err {np.max(np.abs(w-ref))/np.abs(ref).max():.1e} "
              f"res {np.linalg.norm(a@z - z*w)/np.linalg.norm(a):.1e} orth {np.abs(z.T@z-np.eye(n)).max():.1e}", flush=True)
