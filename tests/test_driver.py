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
def test_driver_fkf_matches_oracle(tmp_path, cfg):
    """cmd_run's fkf branch (driver.hpp:278-303) through the shim against the CPU oracle."""
    from oracle import oracle as O
    exe = _build(tmp_path)
    d = E.simulate(str(tmp_path / "exp"), cfg, 3)
    out = str(tmp_path / "out")
    r = subprocess.run([exe, d, out, "fkf"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    w, h, ys, s2 = W.problem(cfg, 3)  # c3: whitened H and y, σ² = 1
    k, p = w.ghep_sizes()
    ocov = O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu)
    of = O.FastFilter(ocov, O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val), s2, k, p, w.ghep_seed)
    for step, y in enumerate(ys, start=1):
        of.step(y)
        _, _, mean = P.read_field(os.path.join(out, f"mean_step{step:03d}.fkf"))
        assert rel_err(mean, of.state()["mean"]) < 1e-9
    rows = open(os.path.join(out, "metrics.csv")).read().splitlines()
    assert rows[0] == "step,wall_time_s,rel_l2_error,effective_rank,trace_criterion,relative_entropy"
    last = rows[-1].split(",")
    assert int(last[0]) == 3 and float(last[3]) == of.rank
    assert abs(float(last[4]) - of.trace_criterion()) <= 1e-9 * abs(of.trace_criterion())
    assert abs(float(last[5]) - of.relative_entropy()) <= 1e-9 * abs(of.relative_entropy())
    fks = P.read_state(os.path.join(out, "state_step003.fks"))
    assert fks["alpha"] == 3.0 and fks["w"].shape == (w.N, of.rank)
    assert rel_err(fks["mean"], of.state()["mean"]) < 1e-9
    assert np.max(np.abs(fks["d"] - of.state()["d"])) / 3.0 < 1e-9


@pytest.mark.gpu
def test_driver_uq_sample_bench_match_oracle(tmp_path):
    """cmd_uq (driver.hpp:368-406), cmd_sample (:411-460, FFT mode) over the FKS1 states of an
    fkf run, and the cmd_bench CSV (:489-616), against the CPU oracle."""
    from oracle import oracle as O
    exe = _build(tmp_path)
    d = E.simulate(str(tmp_path / "exp"), "c0", 3)
    run = str(tmp_path / "run")
    r = subprocess.run([exe, d, run, "fkf", "--states", "all"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for what in ("variance", "trace", "entropy"):
        r = subprocess.run([exe, "uq", run, str(tmp_path / "uq"), what], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "sample", run, str(tmp_path / "smp"), "2", "--steps", "1,3"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    w, h, ys, s2 = W.problem("c0", 3)
    k, p = w.ghep_sizes()
    ocov = O.CovarianceOperator(w.n, w.n, family=1, theta=w.theta, length=w.length, nu=w.nu)
    of = O.FastFilter(ocov, O.Csr.from_arrays(h.rows, h.cols, h.rowptr, h.col, h.val), s2, k, p, w.ghep_seed)
    tr = {int(a): float(b) for a, b in (l.split(",") for l in open(tmp_path / "uq" / "uq_trace.csv").read().split()[1:])}
    en = {int(a): float(b) for a, b in (l.split(",") for l in open(tmp_path / "uq" / "uq_entropy.csv").read().split()[1:])}
    for step, y in enumerate(ys, start=1):
        of.step(y)
        _, _, var = P.read_field(str(tmp_path / "uq" / f"variance_step{step:03d}.fkf"))
        assert rel_err(var, of.variance()) < 1e-9
        assert abs(tr[step] - of.trace_criterion()) <= 1e-9 * abs(of.trace_criterion())
        assert abs(en[step] - of.relative_entropy()) <= 1e-9 * abs(of.relative_entropy())
        if step in (1, 3):
            xo = of.realizations(w.sample_seed, 2)
            mo = of.state()["mean"]
            for j in range(2):
                _, _, x = P.read_field(str(tmp_path / "smp" / f"sample_step{step:03d}_r{j:03d}.fkf"))
                assert rel_err(x - mo, xo[:, j] - mo) < 1e-9
    # cmd_sample refuses enkf runs like the reference (driver.hpp:418-421)
    r = subprocess.run([exe, d, str(tmp_path / "en"), "enkf", "--members", "8"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "sample", str(tmp_path / "en"), str(tmp_path / "x"), "1"], capture_output=True, text=True)
    assert r.returncode == 1 and "do not save" in r.stderr
    csv = str(tmp_path / "bench.csv")
    r = subprocess.run([exe, "bench", d, csv, "32x32,48x40", "fkf"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = open(csv).read().splitlines()
    assert rows[0] == "grid,nx,ny,n_s,kind,offline_s,step_median_s,step_min_s,step_max_s"
    assert [x.split(",")[:5] for x in rows[1:]] == [["32x32", "32", "32", "1024", "fkf"], ["48x40", "48", "40", "1920", "fkf"]]
    for x in rows[1:]:
        off, med, lo, hi = (float(v) for v in x.split(",")[5:])
        assert off > 0 and 0 < lo <= med <= hi


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
