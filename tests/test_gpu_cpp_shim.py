"""The C++ drop-in shim (include/fastkf_b200.hpp) compiled by g++ behaves like the Python
mirror and the oracle: same α, trace, entropy and mean per step (reference driver flow,
driver.hpp:278-303)."""
import os
import subprocess

import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from tests.helpers import Problem, rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1405_2276_b200")


def _compile(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", LIBDIR, "-lfastkf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_shim_compiles_without_gpu(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_cpp_shim_matches_oracle(tmp_path):
    exe = _compile(tmp_path)
    p = Problem(12, 12, 3, 8, 3, 2e-4)
    stdin = "\n".join(" ".join(repr(float(v)) for v in y) for y in p.obs)
    out = subprocess.run([exe, "3"], input=stdin, capture_output=True, text=True, check=True).stdout.split("\n")
    of = O.FastFilter(p.oracle_cov(), p.oracle_h(), p.sigma2, 16, 20, 11)
    i = 0
    for k, y in enumerate(p.obs):
        of.step(y)
        hdr = out[i].split()
        i += 1
        mean = np.array([float(v) for v in out[i:i + 144]])
        i += 144
        assert int(hdr[1]) == k + 1 and float(hdr[3]) == k + 1.0
        assert rel_err(mean, of.state()["mean"]) < 1e-9
        assert abs(float(hdr[5]) - of.trace_criterion()) <= 1e-9 * abs(of.trace_criterion())
        assert abs(float(hdr[7]) - of.relative_entropy()) <= 1e-9 * abs(of.relative_entropy())
    assert out[i].strip() == "edit ok"
    assert out[i + 1].strip() == "run ok"  # fkf_run (the driver loop in one call) ≡ fkf_step × 2


def _compile_fekf(tmp_path):
    exe = str(tmp_path / "shim_fekf_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_fekf_demo.cpp"), "-L", LIBDIR, "-lfastkf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_fekf_shim_compiles_without_gpu(tmp_path):
    assert os.path.exists(_compile_fekf(tmp_path))


@pytest.mark.gpu
def test_cpp_fekf_shim_matches_oracle(tmp_path):
    """cmd_run's ekf branch through the C++ shim (driver.hpp:304-333) against the oracle."""
    from paper_1405_2276_b200 import workloads as W
    from tests.helpers import EXPERIMENT
    exe = _compile_fekf(tmp_path)
    p = Problem(8, 8, 2, 4, 4, 2e-4, kernel=dict(EXPERIMENT, theta=1e-4))
    seeds = [W.derive_seed(905, k) for k in range(4)]
    stdin = "\n".join(" ".join(repr(float(v)) for v in y) + f" {sd}" for y, sd in zip(p.obs, seeds))
    out = subprocess.run([exe, "4"], input=stdin, capture_output=True, text=True, check=True).stdout.split("\n")
    mean0 = np.full(64, O.boxcox(2.0, [1e-4], "forward")[0])
    o = O.ExtendedFilter(p.oracle_cov(), p.oracle_h(), mean0)
    i = 0
    for k, (y, sd) in enumerate(zip(p.obs, seeds)):
        o.step(y, p.sigma2, 2.0, k_rank=p.h.rows, trunc_tol=0.0, seed=sd)
        st = o.state()
        hdr = out[i].split()
        i += 1
        mean = np.array([float(v) for v in out[i:i + 64]])
        i += 64
        assert int(hdr[1]) == k + 1 and float(hdr[3]) == st["alpha"]
        assert int(hdr[5]) == len(st["d"]) and int(hdr[7]) == len(st["d"])
        assert rel_err(mean - mean0, st["mean"] - mean0) < 1e-9
