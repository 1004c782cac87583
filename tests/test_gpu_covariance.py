"""GPU parity: K1 (Γ·X via FFT circulant embedding), K3 (Ω), sampler, K2 (SpMM).

Mirrors proj/tests/test_kernel_covariance.cpp:89-154 and checks every device result
against the CPU oracle on identical inputs."""
import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from tests.helpers import EXPERIMENT, kernel_fn, kernel_matrix, rel_err

pytestmark = pytest.mark.gpu

GRIDS = [(20, 20, 1.0, 1.0), (13, 7, 2.0, 1.0), (64, 64, 1.0, 1.0), (59, 55, 1.0, 1.0), (9, 11, 1.0, 1.0)]


def _pair(nx, ny, lx, ly, kernel):
    g = P.Grid(nx, ny, lx, ly)
    return (P.CovarianceOperator(g, P.KernelSpec(**kernel)),
            O.CovarianceOperator(nx, ny, lx, ly, **kernel))


@pytest.mark.parametrize("nx,ny,lx,ly", GRIDS)
def test_fft_apply_matches_oracle_and_dense(nx, ny, lx, ly):
    gpu, orc = _pair(nx, ny, lx, ly, EXPERIMENT)
    assert (gpu.mx, gpu.my) == (orc.mx, orc.my)
    X = O.gaussian_matrix(nx * ny, 5, 11, 0)
    Yg = gpu.apply(X)
    Yo = orc.apply(X)
    assert rel_err(Yg, Yo) < 1e-12
    if nx * ny <= 4096:  # test_kernel_covariance.cpp:100-109 (dense oracle ≤ 1e-12)
        K = kernel_matrix(nx, ny, kernel_fn(**EXPERIMENT), lx, ly)
        for j in range(3):
            assert rel_err(Yg[:, j], K @ X[:, j]) < 1e-12


def test_one_cell_operator_is_the_sill():  # test_kernel_covariance.cpp:89-98
    g = P.Grid(1, 1)
    cov = P.CovarianceOperator(g, P.KernelSpec(family=0, theta=3e-3, length=0.2, power=0.5))
    assert abs(cov.apply(np.array([2.0]))[0] - 6e-3) <= 1e-13 * 6e-3
    assert abs(cov.trace() - 3e-3) <= 1e-14


def test_columns_and_symmetry():  # test_kernel_covariance.cpp:111-132
    gpu, _ = _pair(9, 11, 1.0, 1.0, EXPERIMENT)
    K = kernel_matrix(9, 11, kernel_fn(**EXPERIMENT))
    for i in (0, 40, 98):
        e = np.zeros(99)
        e[i] = 1.0
        assert rel_err(gpu.apply(e), K[:, i]) < 1e-12
    norm = np.linalg.norm(K, 2)
    for t in range(5):
        x = W.rng_normals(99, 21, 2 * t)
        y = W.rng_normals(99, 21, 2 * t + 1)
        assert abs(gpu.apply(x) @ y - x @ gpu.apply(y)) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(y) * norm
    with pytest.raises(ValueError):
        gpu.apply(np.zeros(5))


def test_spectrum_matches_oracle():
    for nx, ny, lx, ly in GRIDS[:3]:
        gpu, orc = _pair(nx, ny, lx, ly, EXPERIMENT)
        sg, so = gpu.spectrum(), orc.spectrum()
        assert np.max(np.abs(sg - so)) <= 1e-12 * np.max(np.abs(so))
        assert sg.min() >= 0.0


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_baseline_tori_and_apply(name):
    w = W.CONFIGS[name]
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    gpu, orc = _pair(w.n, w.n, 1.0, 1.0, kern)
    assert (gpu.mx, gpu.my) == (orc.mx, orc.my)
    assert gpu.mx == {"c0": 128, "c1": 512, "c2": 512}[name]  # SURVEY.md §0 probe (c1 needs pad 2)
    X = O.gaussian_matrix(w.N, 3, 5, 0)
    assert rel_err(gpu.apply(X), orc.apply(X)) < 1e-12


@pytest.mark.parametrize("nx,ny,lx,ly", GRIDS + [(256, 256, 1.0, 1.0), (128, 96, 1.5, 1.0)])
def test_single_vector_path_matches_batched(nx, ny, lx, ly):
    """The per-step Γ·x path (warp-per-transform kernels) against the batched kernels and the
    oracle on the same vectors."""
    gpu, orc = _pair(nx, ny, lx, ly, EXPERIMENT)
    X = O.gaussian_matrix(nx * ny, 8, 13, 0)
    Yb = gpu.apply(X)
    for j in (0, 5):
        y1 = gpu.apply(np.ascontiguousarray(X[:, j]))
        assert rel_err(y1, Yb[:, j]) < 1e-14
        assert rel_err(y1, orc.apply(np.ascontiguousarray(X[:, j]))) < 1e-12


def test_embedding_failure_names_the_kernel():  # test_kernel_covariance.cpp:304-320
    with pytest.raises(RuntimeError, match="powered-exponential.*theta"):
        P.CovarianceOperator(P.Grid(16, 16), P.KernelSpec(family=0, theta=1.0, length=2.0, power=2.0))
    with pytest.raises(RuntimeError, match="matern.*theta"):
        P.CovarianceOperator(P.Grid(8, 8), P.KernelSpec(family=1, theta=1.0, length=50.0, nu=3.5))


def test_gaussian_matrix_matches_reference_streams():
    g = P.gaussian_matrix(1001, 7, 12345, 3)
    o = O.gaussian_matrix(1001, 7, 12345, 3)
    assert np.max(np.abs(g - o)) < 1e-13  # integer stream exact; libm vs libdevice ≤ few ulp


def test_sample_pair_matches_oracle():
    for nx, ny, lx, ly in GRIDS[:3]:
        gpu, orc = _pair(nx, ny, lx, ly, EXPERIMENT)
        a, b = gpu.sample_pair(99, 3)
        ao, bo = orc.sample_pair(99, 3)
        assert rel_err(a, ao) < 1e-10 and rel_err(b, bo) < 1e-10


@pytest.mark.parametrize("nx,ny", [(512, 8), (8, 512), (512, 64), (64, 512)])
@pytest.mark.parametrize("ncols", [1, 9])
def test_register_resident_1024_passes(nx, ny, ncols):
    """1024-point register transforms in one direction only (the other is a short
    compile-time or generic schedule), single vector and batched, against the oracle."""
    kern = dict(family=1, theta=1.0, length=0.1, nu=0.5)
    gpu = P.CovarianceOperator(P.Grid(nx, ny), P.KernelSpec(**kern))
    orc = O.CovarianceOperator(nx, ny, **kern)
    assert (gpu.mx, gpu.my) == (orc.mx, orc.my) and 1024 in (gpu.mx, gpu.my)
    X = O.gaussian_matrix(nx * ny, ncols, 5, 1)
    Yg = gpu.apply(X if ncols > 1 else X[:, 0]).reshape(nx * ny, -1)
    Yo = np.stack([orc.apply(X[:, j]) for j in range(ncols)], axis=1)
    assert rel_err(Yg, Yo) < 1e-12


@pytest.mark.parametrize("name,ncols", [("c4", 1), ("c4", 9), ("c2", 1), ("c2", 9)])
def test_register_resident_tori_match_oracle(name, ncols):
    """The register-resident transforms: 512² tori (8³ radix-8) and the c4 1024² torus
    (2·8³: a register radix-2 pass, three radix-8 exchanges), single vector (the step's
    Γ(Hᵀz)) and batched (≥ 8 columns: the offline Γ·X), against the oracle's FFTW restatement."""
    w = W.CONFIGS[name]
    kern = dict(family=1, theta=w.theta, length=w.length, nu=w.nu)
    gpu = P.CovarianceOperator(P.Grid(w.n, w.n), P.KernelSpec(**kern))
    orc = O.CovarianceOperator(w.n, w.n, **kern)
    assert (gpu.mx, gpu.my) == (orc.mx, orc.my)
    X = O.gaussian_matrix(w.N, ncols, 17, 3)
    Yg = gpu.apply(X if ncols > 1 else X[:, 0])
    Yo = np.stack([orc.apply(X[:, j]) for j in range(ncols)], axis=1)
    assert rel_err(Yg.reshape(w.N, -1), Yo) < 1e-12
