"""Oracle fkf_init wall time per config on this host (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from tests.helpers import workload_inputs
O.set_threads(os.cpu_count() or 1)
for name in sys.argv[1:]:
    w, h, ys, s2 = workload_inputs(name, 1)
    k, p = w.ghep_sizes()
    t = time.perf_counter()
    ocov = O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu)
    of = O.FastFilter(ocov, O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val), s2, k, p, w.ghep_seed)
    t1 = time.perf_counter()
    of.step(ys[0])
    print(name, f"oracle init {t1 - t:.1f}s, step {time.perf_counter() - t1:.2f}s, cores {os.cpu_count()}", flush=True)
