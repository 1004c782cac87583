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
