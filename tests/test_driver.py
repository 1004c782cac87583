"""The reference-style driver (tools/fkb_run.cpp, the fkf / ekf / enkf branches of cmd_run,
driver.hpp:203-340) over experiment directories written by paper_1405_2276_b200/experiment.py
(cmd_simulate's files, driver.hpp:130-153).  CPU: the writer's formats and the driver build;
GPU: the driver's means against the Python mirror and the oracle, metrics.csv and FKS1."""
import os
import subprocess

import numpy as np
import pytest

import paper_1405_2276_b200 as P
from paper_1405_2276_b200 import experiment as E
from paper_1405_2276_b200 import workloads as W
from tests.helpers import rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1405_2276_b200")


def _build(tmp_path):
    exe = str(tmp_path / "fkb_run")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "fkb_run.cpp"), "-L", LIBDIR, "-lfastkf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_experiment_files_and_driver_build(tmp_path):
    d = E.simulate(str(tmp_path / "exp"), "c0", 2)
    w, h, ys, s2 = W.problem("c0", 2)
    lines = open(os.path.join(d, "observations.csv")).read().splitlines()
    assert lines[0] == "step,measurement,value" and len(lines) == 1 + 2 * w.m
    y1 = np.array([float(l.split(",")[2]) for l in lines[1:1 + w.m]])
    assert np.array_equal(y1, ys[0])  # repr round trip is exact
    nx, ny, t0 = P.read_field(os.path.join(d, "truth_step000.fkf"))
    assert (nx, ny) == (64, 64) and not t0.any()
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c0", "c3"])
def test_driver_fkf_matches_mirror(tmp_path, cfg):
    exe = _build(tmp_path)
    d = E.simulate(str(tmp_path / "exp"), cfg, 3)
    out = str(tmp_path / "out")
    r = subprocess.run([exe, d, out, "fkf"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    w, h, ys, s2 = W.problem(cfg, 3)  # c3: whitened H and y, σ² = 1
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
    k, p = w.ghep_sizes()
    ctx = P.fkf_init(cov, h, s2, k, p, w.ghep_seed)
    for step, y in enumerate(ys, start=1):
        st = P.fkf_step(ctx, y)
        _, _, mean = P.read_field(os.path.join(out, f"mean_step{step:03d}.fkf"))
        assert rel_err(mean, st["mean"]) < 1e-12
    rows = open(os.path.join(out, "metrics.csv")).read().splitlines()
    assert rows[0] == "step,wall_time_s,rel_l2_error,effective_rank,trace_criterion,relative_entropy"
    last = rows[-1].split(",")
    assert int(last[0]) == 3 and float(last[3]) == ctx.rank()
    assert abs(float(last[4]) - ctx.trace_criterion()) <= 1e-12 * abs(ctx.trace_criterion())
    fks = P.read_state(os.path.join(out, "state_step003.fks"))
    assert fks["alpha"] == 3.0 and fks["w"].shape == (w.N, ctx.rank())
    assert rel_err(fks["mean"], st["mean"]) < 1e-12


@pytest.mark.gpu
def test_driver_ekf_and_enkf(tmp_path):
    exe = _build(tmp_path)
    d = E.simulate(str(tmp_path / "exp"), "c0", 2)
    w, h, ys, s2 = W.problem("c0", 2)
    cov = P.CovarianceOperator(P.Grid(w.n, w.n), W.kernel_spec(w))
    k, p = w.ghep_sizes()
    out = str(tmp_path / "ekf")
    r = subprocess.run([exe, d, out, "ekf"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    g = P.ExtendedFilter(cov, h, np.full(w.N, -1.0))  # Box–Cox 1, init 0: mean0 = forward(0) = −1
    for step, y in enumerate(ys, start=1):
        g.step(y, s2, P.BoxCox(1.0), P.FekfOptions(k_rank=k, oversampling=p, trunc_tol=1e-5,
                                                     seed=W.derive_seed(w.seed, 4000 + step)))
        _, _, mean = P.read_field(os.path.join(out, f"mean_step{step:03d}.fkf"))
        assert rel_err(mean, g.state(with_w=False)["mean"] + 1.0) < 1e-12
    assert P.read_state(os.path.join(out, "state_step002.fks"))["w"].shape[1] == g.rank()
    last = open(os.path.join(out, "metrics.csv")).read().splitlines()[-1].split(",")
    assert abs(float(last[4]) - g.trace_criterion()) <= 1e-12 * abs(g.trace_criterion())
    assert abs(float(last[5]) - g.relative_entropy()) <= 1e-12 * abs(g.relative_entropy())
    out = str(tmp_path / "enkf")
    r = subprocess.run([exe, d, out, "enkf", "--members", "64"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    ens = P.Ensemble(cov, h, 64)
    for step, y in enumerate(ys, start=1):
        ens.step(y, s2, W.derive_seed(w.seed, 2000 + step))
        _, _, mean = P.read_field(os.path.join(out, f"mean_step{step:03d}.fkf"))
        assert rel_err(mean, ens.mean()) < 1e-13
