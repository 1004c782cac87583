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

from tests.parity import run_config, run_config_batch  # noqa: E402


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
    # per-call steps, then the same configs as ONE batch call (fkb_fkf_run / fkb_fkf_run_uq), as
    # the default full step graphs and as the opt-in pipelined graphs (FKB_PIPED=1)
    jobs = [("per_call", c, s) for c, s in runs]
    jobs += [(mode, c, 1) for mode in ("batch", "batch_piped") for c in a.configs.split(",") if c]
    for mode, cfg, solver in jobs:
        t0 = time.perf_counter()
        if mode == "per_call":
            res = run_config(cfg, solver=solver)
        else:
            os.environ["FKB_PIPED"] = "1" if mode == "batch_piped" else "0"
            res = run_config_batch(cfg)
            os.environ.pop("FKB_PIPED", None)
        res["mode"] = mode
        res["wall_s"] = time.perf_counter() - t0
        results.append(res)
        print(json.dumps({"mode": mode, "config": cfg, "solver": solver, "worst": res["worst"],
                          "wall_s": res["wall_s"]}), flush=True)
        with open(a.out, "w") as f:
            json.dump({"tolerance": 1e-9, "norms": "mean/var: ||d||2/||ref||2; d: max|dd|/alpha; lambda: "
                       "max|dl|/l1 and per-eigenvalue over l_i >= 1e-3 l1; realizations: ||dx||/||x_ref-mean||",
                       "runs": results}, f, indent=1)


if __name__ == "__main__":
    main()
