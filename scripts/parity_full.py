"""Record full-length GPU-vs-oracle parity for the BASELINE configs (per-step worst errors)
into a JSON file (default profiles/parity_r02.json).  Usage:
    python scripts/parity_full.py [--configs c0,c1,c2,c3,c4] [--solvers 1] [--out PATH]
Test infrastructure: it imports the oracle as the checker (tests/parity.py)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.parity import run_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
    ap.add_argument("--solvers", default="1")
    ap.add_argument("--extra", default="c1:0,c2:0", help="config:solver pairs run in addition")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r02.json"))
    a = ap.parse_args()
    runs = [(c, int(s)) for c in a.configs.split(",") if c for s in a.solvers.split(",")]
    runs += [(c, int(s)) for c, s in (x.split(":") for x in a.extra.split(",") if x)]
    results = []
    for cfg, solver in runs:
        t0 = time.perf_counter()
        res = run_config(cfg, solver=solver)
        res["wall_s"] = time.perf_counter() - t0
        results.append(res)
        print(json.dumps({"config": cfg, "solver": solver, "worst": res["worst"], "wall_s": res["wall_s"]}), flush=True)
        with open(a.out, "w") as f:
            json.dump({"tolerance": 1e-9, "norms": "mean/var: ||d||2/||ref||2; d: max|dd|/alpha; lambda: "
                       "max|dl|/l1 and per-eigenvalue over l_i >= 1e-3 l1; realizations: ||dx||/||x_ref-mean||",
                       "runs": results}, f, indent=1)


if __name__ == "__main__":
    main()
