"""FKF1 / FKS1 snapshot formats (field_io.hpp:18-135) through the Python mirror and the C++
shim, restating proj/tests/test_cli_io.cpp:61-100 and pinning the byte layout.  CPU."""
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_1405_2276_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1405_2276_b200")


def test_field_round_trip_and_layout(tmp_path):  # test_cli_io.cpp:61-69
    data = np.random.default_rng(5).standard_normal(84)
    P.write_field(tmp_path / "f.fkf", 12, 7, data)
    raw = (tmp_path / "f.fkf").read_bytes()
    assert raw[:4] == b"FKF1" and struct.unpack("<II", raw[4:12]) == (12, 7) and len(raw) == 12 + 8 * 84
    nx, ny, back = P.read_field(tmp_path / "f.fkf")
    assert (nx, ny) == (12, 7) and np.array_equal(back, data)


def test_field_reader_rejects_corrupt(tmp_path):  # test_cli_io.cpp:71-83
    (tmp_path / "bad.fkf").write_bytes(b"NOPE----------------")
    with pytest.raises(RuntimeError, match="not a FKF1"):
        P.read_field(tmp_path / "bad.fkf")
    P.write_field(tmp_path / "t.fkf", 4, 4, np.ones(16))
    (tmp_path / "t.fkf").write_bytes((tmp_path / "t.fkf").read_bytes()[:40])
    with pytest.raises(RuntimeError, match="truncated"):
        P.read_field(tmp_path / "t.fkf")
    with pytest.raises(FileNotFoundError):
        P.read_field(tmp_path / "missing.fkf")
    with pytest.raises(ValueError, match="does not match 3x3"):
        P.write_field(tmp_path / "x.fkf", 3, 3, np.ones(5))


def test_state_round_trip_and_layout(tmp_path):  # test_cli_io.cpp:85-100
    rng = np.random.default_rng(6)
    st = {"alpha": 3.0, "step": 3, "mean": rng.standard_normal(20), "d": np.linspace(0.1, 0.9, 4),
          "w": rng.standard_normal((20, 4))}
    P.write_state(tmp_path / "s.fks", st)
    raw = (tmp_path / "s.fks").read_bytes()
    assert raw[:4] == b"FKS1" and struct.unpack("<IIId", raw[4:24]) == (20, 4, 3, 3.0)
    assert np.array_equal(np.frombuffer(raw, "<f8", 80, 24 + 8 * 24).reshape(4, 20).T, st["w"])  # column-major W
    back = P.read_state(tmp_path / "s.fks")
    for k in ("alpha", "step"):
        assert back[k] == st[k]
    for k in ("mean", "d", "w"):
        assert np.array_equal(back[k], st[k])


def test_cpp_shim_io_matches_python(tmp_path):
    exe = str(tmp_path / "io_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_io_demo.cpp"), "-L", LIBDIR, "-lfastkf_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    out = subprocess.run([exe, str(tmp_path / "c.fkf"), str(tmp_path / "c.fks")], capture_output=True, text=True)
    assert out.returncode == 0 and "io ok" in out.stdout, (out.returncode, out.stderr)
    nx, ny, data = P.read_field(tmp_path / "c.fkf")
    i = np.arange(84)
    assert (nx, ny) == (12, 7) and np.array_equal(data, 0.25 * i - 3.0 + 1e-3 * (i * i))
    st = P.read_state(tmp_path / "c.fks")
    w = (np.arange(20)[:, None] + 1.0) / (np.arange(4)[None, :] + 2.0)
    assert st["alpha"] == 3.0 and st["step"] == 3 and np.array_equal(st["w"], w)
