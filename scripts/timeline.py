"""Device timeline of graph-replayed filter steps (CUPTI through torch.profiler): every kernel's
start/end relative to the step's first kernel, per stream — shows the real critical path
(the event-marked in-graph phase times include event-node overhead).  Development aid.

    python scripts/timeline.py [c2] [steps] [batch]     (batch: one steps_async call of `steps` steps)
"""
import sys, os, json, tempfile
sys.path = [p for p in sys.path if os.path.abspath(p or '.') != os.path.dirname(os.path.abspath(__file__))]  # scripts/profile.py shadows the stdlib module
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1405_2276_b200 as P
from paper_1405_2276_b200._native import DeviceArray, lib, check
from tests.helpers import workload_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
batch = len(sys.argv) > 3 and sys.argv[3] == "batch"
w, h, ys, s2 = workload_inputs(name)
cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(family=1, theta=w.theta, length=w.length, nu=w.nu))
k, p = w.ghep_sizes()
ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
dys = DeviceArray.from_host(np.stack(ys).ravel())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx.steps_async(dys.ptr, 3, w.m)
ctx.sync(3)
check(lib().fkb_dsync())
from torch.profiler import profile, ProfilerActivity
if batch:
    ctx.steps_async(dys.ptr, nsteps, w.m)
    ctx.sync(nsteps)
    check(lib().fkb_dsync())
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if batch:  # the pipelined batch: one flush, then every graph back to back
        flush.zero_()
        torch.cuda.synchronize()
        ctx.steps_async(dys.ptr, nsteps, w.m)
        check(lib().fkb_dsync())
    for i in range(0 if batch else nsteps):
        flush.zero_()
        torch.cuda.synchronize()
        ctx.steps_async(dys.ptr, 1, w.m)
        check(lib().fkb_dsync())
ctx.sync(nsteps)
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
steps, cur = [], None
for e in ev:
    if "elementwise" in e["name"] or "vectorized" in e["name"] or "fill" in e["name"].lower():
        cur = []
        steps.append(cur)
        continue
    if cur is not None:
        cur.append(e)
short = lambda s: s.split("(")[0].replace("void ", "")[:48]
if batch:  # one timeline: every kernel of the batch from the third prologue on
    st = steps[0]
    pro = [i for i, e in enumerate(st) if "k_step_prologue" in e["name"]]
    lo = pro[2] if len(pro) > 4 else 0
    hi = pro[4] if len(pro) > 4 else len(st)
    t0 = st[lo]["ts"]
    print(f"batch: {len(pro)} steps in {(st[-1]['ts'] + st[-1]['dur'] - st[0]['ts']):.1f} us; "
          f"prologue to prologue: {[round(st[b]['ts'] - st[a]['ts'], 1) for a, b in zip(pro, pro[1:])]}")
    for e in st[lo:hi]:
        print(f"  s{e['args'].get('stream', '?'):>3}  {e['ts'] - t0:7.1f} → {e['ts'] + e['dur'] - t0:7.1f}  "
              f"({e['dur']:5.1f})  {short(e['name'])}")
    sys.exit(0)
for si, st in enumerate(steps):
    if not st:
        continue
    t0 = st[0]["ts"]
    end = max(e["ts"] + e["dur"] for e in st)
    print(f"step {si}: {end - t0:.1f} us, {len(st)} kernels")
    if si == len(steps) - 1 or si == 1:
        for e in st:
            print(f"  s{e['args'].get('stream', '?'):>3}  {e['ts'] - t0:7.1f} → {e['ts'] + e['dur'] - t0:7.1f}  "
                  f"({e['dur']:5.1f})  {short(e['name'])}")
