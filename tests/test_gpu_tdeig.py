"""The GPU symmetric eigensolver of the GHEP core T and the add_low_rank core M (tdeig.cu:
Householder tridiagonalization (cluster-resident up to n ≈ 660, grid-wide beyond) and Q on the
GPU, QL rotations applied on the GPU), the
SelfAdjointEigenSolver calls of lowrank.hpp:193, :265-270, against numpy's eigh."""
import numpy as np
import pytest

from paper_1405_2276_b200 import fastkf as F

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 64, 320, 600, 640, 700])
@pytest.mark.parametrize("graded", [False, True])
def test_tridiag_eig_matches_eigh(n, graded):
    rng = np.random.default_rng(n + (1000 if graded else 0))
    if graded:  # the GHEP/core spectra span many decades, with a few negative entries
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.logspace(-8, 6, n) * np.where(rng.random(n) < 0.1, -1.0, 1.0)
        a = (q * lam) @ q.T
    else:
        a = rng.standard_normal((n, n))
    a = 0.5 * (a + a.T)
    w, z = F.sym_eig_tridiag(a)
    wr = np.linalg.eigvalsh(a)
    scale = max(np.abs(wr).max(), 1e-300)
    assert np.all(np.diff(w) >= 0)
    assert np.max(np.abs(w - wr)) <= 1e-13 * scale * max(1, np.sqrt(n) / 4)
    assert np.linalg.norm(a @ z - z * w) <= 1e-13 * np.linalg.norm(a) * max(1.0, np.sqrt(n) / 4)
    assert np.abs(z.T @ z - np.eye(n)).max() <= 1e-12


def test_tridiag_eig_diagonal_and_repeated():
    a = np.diag([3.0, -1.0, 3.0, 0.0, 2.0])
    w, z = F.sym_eig_tridiag(a)
    assert np.allclose(w, [-1.0, 0.0, 2.0, 3.0, 3.0], rtol=0, atol=1e-15)
    assert np.abs(z.T @ z - np.eye(5)).max() <= 1e-14
    assert np.linalg.norm(a @ z - z * w) <= 1e-14
