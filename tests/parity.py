"""Full-length parity of the GPU fast filter against the CPU oracle (test infrastructure).

One BASELINE config is run through the product (C ABI via the Python mirror) and through the
oracle's restatement of fkf_init / fkf_step (fast_filter.hpp:51-125) on byte-identical inputs,
step by step, recording the SURVEY.md §8(c) parity norms per step:

* mean: ‖Δ‖₂/‖ref‖₂ (oracles.hpp:79-81 convention);
* d: max|Δd|/α_k;  α: exact;
* λ (once, after fkf_init): normwise max|Δλ|/λ₁ and the per-eigenvalue relative error over
  λᵢ ≥ 1e-3·λ₁;
* diag Σ (uq.hpp:16-23): ‖Δ‖₂/‖ref‖₂;
* realizations (App. A.4, identical circulant noise): ‖Δ‖₂/‖x_ref − mean_ref‖₂.

Used by tests/test_gpu_parity_full.py (asserts ≤ 1e-9 on every step) and by
scripts/parity_full.py (writes profiles/parity_r02.json)."""
from __future__ import annotations

import time

import numpy as np

from tests.helpers import rel_err, workload_inputs

TOL = 1e-9
STEPS = {"c0": 10, "c1": 20, "c2": 30, "c3": 30, "c4": 50}
UQ = {"c0": True, "c1": True, "c2": False, "c3": True, "c4": True}
REALIZATIONS = {"c0": 2, "c3": 8}


def lambda_errors(lam, lo):
    lam, lo = np.asarray(lam), np.asarray(lo)
    normwise = float(np.max(np.abs(lam - lo)) / lo[0]) if len(lo) else 0.0
    sel = lo >= 1e-3 * lo[0] if len(lo) else np.zeros(0, bool)
    per = float(np.max(np.abs(lam[sel] - lo[sel]) / lo[sel])) if sel.any() else 0.0
    return normwise, per, int(sel.sum())


_ORACLE_CACHE = {}


def oracle_trajectory(name, steps, uq, realizations):
    """The oracle's fkf_init + `steps` fkf_step calls on the config's inputs, every step's state
    (and diag Σ / realizations when asked) kept — computed once per process and shared by the
    per-call, batch and pipelined-batch comparisons (c4's 50 oracle steps take minutes)."""
    from oracle import oracle as O

    key = (name, steps)
    tr = _ORACLE_CACHE.get(key)
    if tr is not None and (tr["uq"] or not uq) and tr["realizations"] >= realizations:
        return tr
    w, h, ys, s2 = workload_inputs(name, steps)
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    t0 = time.perf_counter()
    ocov = O.CovarianceOperator(w.n, w.n, **kern)
    oh = O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val)
    of = O.FastFilter(ocov, oh, s2, k, p, w.ghep_seed)
    tr = dict(init_s=time.perf_counter() - t0, lam=np.array(of.context()["lam"]), rank=int(of.rank), uq=uq,
              realizations=realizations, states=[], var=[], real=[])
    for y in ys:
        of.step(y)
        so = of.state()
        tr["states"].append(dict(alpha=so["alpha"], d=np.array(so["d"]), mean=np.array(so["mean"])))
        if uq:
            tr["var"].append(np.array(of.variance()))
        if realizations:
            tr["real"].append(np.array(of.realizations(w.sample_seed, realizations)))
    _ORACLE_CACHE[key] = tr
    return tr


def run_config(name, steps=None, solver=1, uq=None, realizations=None, record=None):
    """Run `steps` (default: the config's full count) steps on both sides; returns a dict with
    the λ errors and per-step error lists.  `record(dict)` is called after every step."""
    import paper_1405_2276_b200 as P

    steps = STEPS[name] if steps is None else steps
    uq = UQ[name] if uq is None else uq
    realizations = REALIZATIONS.get(name, 0) if realizations is None else realizations
    w, h, ys, s2 = workload_inputs(name, steps)
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    t0 = time.perf_counter()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(**kern))
    ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    ctx.set_solver(solver)
    t_gpu_init = time.perf_counter() - t0
    tr = oracle_trajectory(name, steps, uq, realizations)
    lo = tr["lam"]
    lam_norm, lam_per, lam_n = lambda_errors(ctx.lam, lo)
    out = dict(config=name, solver=solver, steps=steps, rank=int(ctx.rank()), oracle_rank=tr["rank"],
               lambda_normwise=lam_norm, lambda_per_eigenvalue=lam_per, lambda_per_eigenvalue_count=lam_n,
               alpha_exact=True, mean=[], d=[], var=[], real=[], cap_iterations=[], cap_fallback=[],
               gpu_init_s=t_gpu_init, oracle_init_s=tr["init_s"])
    for t, y in enumerate(ys):
        st = P.fkf_step(ctx, y)
        so = tr["states"][t]
        if st["alpha"] != so["alpha"]:
            out["alpha_exact"] = False
        out["mean"].append(rel_err(st["mean"], so["mean"]))
        out["d"].append(float(np.max(np.abs(st["d"] - so["d"])) / so["alpha"]) if len(so["d"]) else 0.0)
        if solver == 1:
            it, fb = ctx.cap_stats()
            out["cap_iterations"].append(int(it))
            out["cap_fallback"].append(bool(fb))
        if uq:
            out["var"].append(rel_err(ctx.variance(), tr["var"][t]))
        if realizations:
            xg = ctx.realizations(w.sample_seed, realizations)
            xo = tr["real"][t]
            out["real"].append(max(rel_err(xg[:, j] - so["mean"], xo[:, j] - so["mean"]) for j in range(realizations)))
        if record:
            record(out)
    out["worst"] = {key: (max(out[key]) if out[key] else 0.0) for key in ("mean", "d", "var", "real")}
    out["worst"]["lambda_normwise"] = lam_norm
    out["worst"]["lambda_per_eigenvalue"] = lam_per
    return out


def run_config_batch(name, steps=None, fused_uq=None):
    """The same comparison with the GPU side run as ONE call over all steps (fkb_fkf_run /
    fkb_fkf_run_uq; with FKB_PIPED=1 the pipelined batch: step t's mean side beside step t+1's
    chain).  With fused_uq the per-step diag Σ and realizations come from the batch's fused pass."""
    import paper_1405_2276_b200 as P

    steps = STEPS[name] if steps is None else steps
    nreal = REALIZATIONS.get(name, 0)
    fused_uq = (name == "c3") if fused_uq is None else fused_uq
    w, h, ys, s2 = workload_inputs(name, steps)
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    k, p = w.ghep_sizes()
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(**kern))
    ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    tr = oracle_trajectory(name, steps, fused_uq or UQ[name], nreal)
    g = ctx.run(np.asarray(ys), count=nreal, seed=w.sample_seed) if fused_uq else ctx.run(np.asarray(ys))
    out = dict(config=name, solver=1, steps=steps, rank=int(ctx.rank()), oracle_rank=tr["rank"], alpha_exact=True,
               mean=[], d=[], var=[], real=[], api="fkb_fkf_run_uq" if fused_uq else "fkb_fkf_run")
    for t in range(len(ys)):
        so = tr["states"][t]
        if g["alpha"][t] != so["alpha"]:
            out["alpha_exact"] = False
        out["mean"].append(rel_err(g["mean"][t], so["mean"]))
        out["d"].append(float(np.max(np.abs(g["d"][t] - so["d"])) / so["alpha"]) if len(so["d"]) else 0.0)
        if fused_uq:
            out["var"].append(rel_err(g["var"][t], tr["var"][t]))
            if nreal:
                xo = tr["real"][t]
                out["real"].append(max(rel_err(g["x"][t, j] - so["mean"], xo[:, j] - so["mean"]) for j in range(nreal)))
    # the state the batch leaves behind is the last step's
    st = ctx.state()
    out["final_state"] = rel_err(st["mean"], tr["states"][-1]["mean"])
    out["worst"] = {key: (max(out[key]) if out[key] else 0.0) for key in ("mean", "d", "var", "real")}
    out["worst"]["final_state"] = out["final_state"]
    return out


def assert_parity(res, tol=TOL):
    assert res["rank"] == res["oracle_rank"], res
    assert res["alpha_exact"], res
    for key, v in res["worst"].items():
        assert v < tol, (key, v, res["config"], res["solver"])
