"""The reference driver's own fkf code (cmd_run's fkf branch, driver.hpp:278-303, and the
cmd_uq loop, :394-406) compiled with g++ against the drop-in shim (include/fastkf_b200.hpp)
and run on BASELINE c0: per-step means, trace and entropy, the FKS1 states it writes, the
cmd_uq variance/trace/entropy recomputed from those files, the standalone randomized_ghep and
RealizationPropagator::at in FFT mode — all against the CPU oracle within 1e-9."""
import os
import subprocess

import numpy as np
import pytest

import paper_1405_2276_b200 as P
from paper_1405_2276_b200 import workloads as W
from tests.helpers import rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1405_2276_b200")
TOL = 1e-9


def _compile(tmp_path):
    exe = str(tmp_path / "driver_verbatim")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "driver_verbatim.cpp"), "-L", LIBDIR, "-lfastkf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_driver_verbatim_compiles_without_gpu(tmp_path):
    assert os.path.exists(_compile(tmp_path))


def _write_inputs(d, w, h, ys, s2):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "problem.txt"), "w") as f:
        f.write(f"{w.n} {w.n} 1 {w.theta!r} {w.length!r} {w.nu!r} {s2!r} {w.seed} {w.rank} {w.oversampling} {len(ys)}\n")
    with open(os.path.join(d, "h.txt"), "w") as f:
        f.write(f"{h.rows} {h.cols} {h.nnz}\n")
        f.write(" ".join(str(int(v)) for v in h.rowptr) + "\n")
        f.write(" ".join(str(int(v)) for v in h.col) + "\n")
        f.write(" ".join(repr(float(v)) for v in h.val) + "\n")
    with open(os.path.join(d, "obs.txt"), "w") as f:
        for y in ys:
            f.write(" ".join(repr(float(v)) for v in y) + "\n")


def _csv(path):
    rows = [l.strip().split(",") for l in open(path).read().strip().splitlines()[1:]]
    return {int(r[0]): [float(x) for x in r[1:]] for r in rows}


@pytest.mark.gpu
def test_driver_fkf_branch_and_cmd_uq_match_oracle(tmp_path):
    from oracle import oracle as O
    exe = _compile(tmp_path)
    w, h, ys, s2 = W.problem("c0")
    inp, out = str(tmp_path / "in"), str(tmp_path / "out")
    _write_inputs(inp, w, h, ys, s2)
    r = subprocess.run([exe, inp, out], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    ocov = O.CovarianceOperator(w.n, w.n, **kern)
    oh = O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val)
    k, p = w.ghep_sizes()
    of = O.FastFilter(ocov, oh, s2, k, p, w.ghep_seed)
    metrics = _csv(os.path.join(out, "metrics.csv"))
    uq_trace = _csv(os.path.join(out, "uq", "uq_trace.csv"))
    uq_ent = _csv(os.path.join(out, "uq", "uq_entropy.csv"))
    for step, y in enumerate(ys, start=1):
        of.step(y)
        so = of.state()
        mean = P.read_field(os.path.join(out, f"mean_step{step:03d}.fkf"))[2]
        assert rel_err(mean, so["mean"]) < TOL
        st = P.read_state(os.path.join(out, f"state_step{step:03d}.fks"))
        assert st["alpha"] == so["alpha"] and st["step"] == step
        assert np.max(np.abs(st["d"] - so["d"])) / so["alpha"] < TOL
        tr, ent = of.trace_criterion(), of.relative_entropy()
        assert abs(metrics[step][0] - tr) <= TOL * abs(tr)
        assert abs(metrics[step][1] - ent) <= TOL * abs(ent)
        assert metrics[step][2] == of.rank
        # cmd_uq on the saved FKS1 states (W read from the file, GPU variance/column norms)
        assert abs(uq_trace[step][0] - tr) <= TOL * abs(tr)
        assert abs(uq_ent[step][0] - ent) <= TOL * abs(ent)
        var = P.read_field(os.path.join(out, "uq", f"variance_step{step:03d}.fkf"))[2]
        assert rel_err(var, of.variance()) < TOL
    # RealizationPropagator::at on the final state, draws 0..2 of sample_seed
    xo = of.realizations(w.sample_seed, 3)
    so = of.state()
    for j in range(3):
        x = P.read_field(os.path.join(out, f"sample_r{j:03d}.fkf"))[2]
        assert rel_err(x - so["mean"], xo[:, j] - so["mean"]) < TOL
    # standalone randomized_ghep
    lam = np.loadtxt(os.path.join(out, "ghep_lambda.txt"))
    lo = of.context()["lam"]
    assert len(lam) == len(lo) and np.max(np.abs(lam - lo)) / lo[0] < TOL
