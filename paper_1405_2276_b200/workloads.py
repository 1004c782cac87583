"""BASELINE.json configurations c0–c4 and their seeded synthetic inputs.

Input generation only (not the hot path, never timed).  Both bench arms and the parity
tests consume the byte-identical arrays produced here: the grid, kernel, ray layout,
σ², rank cap, and per-step observations y_k.

Interpretations of BASELINE.json that the reference API does not cover (SURVEY.md
App. A) are recorded in ``Workload.notes`` and echoed into the bench JSON line:

* truth fields: c0/c1/c4 are a centred Gaussian plume of amplitude 0.5 whose width is
  0.02·k (c4: 0.005·k) at step k, plus 0.1·Σ_{j≤k} w_j with w_j ~ N(0, Γ) circulant
  draws (numpy PCG64 seeded with derive_seed(seed, 6000)); c2/c3 are two drifting
  Gaussian plumes (amplitudes 0.5/0.3, widths 0.08/0.06, starting at (0.30, 0.50) and
  (0.50, 0.70), drifting (+0.01, 0) and (0, −0.01) per step).  The public tomography
  data of the paper (Frio-II) is not used — the configs are synthetic by definition.
* ray layouts: cross_well (tomography.hpp:98-113) for c0/c1/c4; c2/c3 stack a
  left→right 32×32 block and a top→bottom 32×32 block (m = 2048).
* observations: y_k = H s_k + σ·n_k with n_k = gaussian_vector(m, derive_seed(seed,
  1000+k)) exactly as simulate_observations (tomography.hpp:198-211) / obs_seed
  (driver.hpp:77-79).
* c3 per-ray noise: σ_i = 0.002 + 0.018·u_i, u_i = Rng(derive_seed(seed, 6500)).uniform();
  exact whitening H̃ = diag(1/σ_i)H, ỹ = y/σ_i, σ² = 1.
* GHEP sizes follow cmd_run (driver.hpp:281-285): l = min(k+20, N), k = min(k, l),
  p = l − k, ghep seed = derive_seed(seed, 3000).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


# ----------------------------------------------------------------------------- rng.hpp restated (numpy)
def splitmix64(x: int) -> int:
    """rng.hpp:12-18 on Python ints."""
    x = (x + GOLDEN) & MASK
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def derive_seed(seed: int, tag: int) -> int:
    """rng.hpp:22-24."""
    return splitmix64((seed ^ splitmix64(tag)) & MASK)


def _mix_u64(state: np.ndarray) -> np.ndarray:
    z = state
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def rng_uniforms(n: int, seed: int, stream: int = 0) -> np.ndarray:
    """First n Rng(seed, stream).uniform() values (rng.hpp:34-46), counter-addressed."""
    s0 = np.uint64(derive_seed(seed, stream))
    with np.errstate(over="ignore"):
        t = np.arange(1, n + 1, dtype=np.uint64)
        z = _mix_u64(s0 + t * np.uint64(GOLDEN))
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def rng_normals(n: int, seed: int, stream: int = 0) -> np.ndarray:
    """First n Rng(seed, stream).normal() values (rng.hpp:49-61): Box–Muller, cos then sin."""
    npairs = (n + 1) // 2
    u = rng_uniforms(2 * npairs, seed, stream)
    u1, u2 = u[0::2], u[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = (2.0 * math.pi) * u2
    out = np.empty(2 * npairs)
    out[0::2] = rad * np.cos(ang)
    out[1::2] = rad * np.sin(ang)
    return out[:n]


# ----------------------------------------------------------------------------- configs
@dataclasses.dataclass
class Workload:
    name: str
    n: int                 # grid is n×n on the unit square
    nu: float              # Matérn smoothness
    length: float          # correlation length
    theta: float
    sigma2: float          # scalar noise variance passed to fkf_init (1.0 when whitened)
    noise_std: float | None  # homogeneous noise std (None: per-ray, c3)
    steps: int
    rank: int
    seed: int
    layout: str            # "lr" or "lr+tb"
    n_src: int
    truth: str             # "plume_grow" or "two_plumes"
    plume_growth: float = 0.02
    variance_each_step: bool = False
    realizations_per_step: int = 0
    oversampling: int = 20

    @property
    def N(self):
        return self.n * self.n

    @property
    def m(self):
        return self.n_src * self.n_src * (2 if self.layout == "lr+tb" else 1)

    def ghep_sizes(self):
        """(k, p) as cmd_run computes them (driver.hpp:281-285)."""
        l_max = min(self.rank + self.oversampling, self.N)
        k = min(self.rank, l_max)
        return k, l_max - k

    @property
    def ghep_seed(self):
        return derive_seed(self.seed, 3000)  # driver.hpp:83

    @property
    def sample_seed(self):
        return derive_seed(self.seed, 5000)  # driver.hpp:87


CONFIGS = {
    "c0": Workload("c0", 64, 0.5, 0.2, 1.0, 1e-4, 0.01, 10, 256, 0, "lr", 16, "plume_grow", 0.02),
    "c1": Workload("c1", 128, 1.5, 0.15, 1.0, 1e-4, 0.01, 20, 200, 1, "lr", 32, "plume_grow", 0.02,
                   variance_each_step=True),
    "c2": Workload("c2", 256, 0.5, 0.1, 1.0, 2.5e-5, 0.005, 30, 300, 2, "lr+tb", 32, "two_plumes"),
    "c3": Workload("c3", 256, 2.5, 0.05, 1.0, 1.0, None, 30, 400, 3, "lr+tb", 32, "two_plumes",
                   variance_each_step=True, realizations_per_step=8),
    "c4": Workload("c4", 512, 0.5, 0.08, 1.0, 2.5e-5, 0.005, 50, 500, 4, "lr", 64, "plume_grow", 0.005),
}


def layout_points(w: Workload):
    """Source/receiver coordinates; rows of H are source-major per block (tomography.hpp:135-142)."""
    n = w.n_src
    lx = ly = 1.0
    blocks = [(np.array([[0.0, (i + 0.5) * ly / n] for i in range(n)]),
               np.array([[lx, (j + 0.5) * ly / n] for j in range(n)]))]  # cross_well :107-110
    if w.layout == "lr+tb":
        blocks.append((np.array([[(i + 0.5) * lx / n, ly] for i in range(n)]),
                       np.array([[(j + 0.5) * lx / n, 0.0] for j in range(n)])))
    return blocks


def cell_centers(n: int):
    c = (np.arange(n) + 0.5) * (1.0 / n)
    cx, cy = np.meshgrid(c, c, indexing="ij")  # flat index ix*ny + iy (grid.hpp:48)
    return cx.ravel(), cy.ravel()


def _matern(nu, length, theta, r):
    from scipy.special import gamma, kv
    a = math.sqrt(2.0 * nu) * r / length
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        v = theta * 2.0 ** (1.0 - nu) / gamma(nu) * a ** nu * kv(nu, a)
    v = np.where(r == 0.0, theta, v)
    return np.where(a > 700.0, 0.0, v)


def _circulant_sampler(w: Workload):
    """numpy circulant-embedding N(0,Γ) sampler for truth increments (input generation only)."""
    n = w.n
    base = 2 * n - 1
    for pad in (1, 2, 4, 8):
        mx = 1 << (base * pad - 1).bit_length()  # power of two ≥ base·pad (next_smooth subset)
        d = np.minimum(np.arange(mx), mx - np.arange(mx)) * (1.0 / n)
        r = np.hypot(d[:, None], d[None, :])
        lam = np.fft.fft2(_matern(w.nu, w.length, w.theta, r)).real
        if lam.min() >= -1e-10 * lam.max():
            break
    amp = np.sqrt(np.maximum(lam, 0.0) / lam.size)

    def draw(rng):
        z = rng.standard_normal((mx, mx)) + 1j * rng.standard_normal((mx, mx))
        f = np.fft.fft2(amp * z)
        return f.real[:n, :n].ravel().copy()

    return draw


def truth_fields(w: Workload):
    cx, cy = cell_centers(w.n)
    out = []
    if w.truth == "plume_grow":
        rng = np.random.default_rng(derive_seed(w.seed, 6000))
        draw = _circulant_sampler(w)
        acc = np.zeros(w.N)
        for k in range(1, w.steps + 1):
            sig = w.plume_growth * k
            plume = 0.5 * np.exp(-0.5 * ((cx - 0.5) ** 2 + (cy - 0.5) ** 2) / sig ** 2)
            acc += 0.1 * draw(rng)
            out.append(plume + acc)
    else:
        for k in range(1, w.steps + 1):
            a = 0.5 * np.exp(-0.5 * ((cx - (0.30 + 0.01 * k)) ** 2 + (cy - 0.50) ** 2) / 0.08 ** 2)
            b = 0.3 * np.exp(-0.5 * ((cx - 0.50) ** 2 + (cy - (0.70 - 0.01 * k)) ** 2) / 0.06 ** 2)
            out.append(a + b)
    return out


def csr_matvec(rowptr, col, val, x):
    rows = len(rowptr) - 1
    prod = val * x[col]
    out = np.add.reduceat(prod, rowptr[:-1]) if len(prod) else np.zeros(rows)
    out[np.diff(rowptr) == 0] = 0.0
    return out


def per_ray_std(w: Workload):
    u = rng_uniforms(w.m, derive_seed(w.seed, 6500), 0)
    return 0.002 + 0.018 * u


def make_inputs(w: Workload, H, steps: int | None = None):
    """Per-step observations for H = (rowptr, col, val) of the *unwhitened* operator.

    Returns (H_used, ys, sigma2): for c3 H_used is the whitened operator and ys whitened.
    """
    rowptr, col, val = (np.asarray(a) for a in H)
    steps = w.steps if steps is None else steps
    truths = truth_fields(w)[:steps]
    if w.noise_std is None:
        sd = per_ray_std(w)
    else:
        sd = np.full(w.m, w.noise_std)
    ys = []
    for k, s in enumerate(truths, start=1):
        noise = rng_normals(w.m, derive_seed(w.seed, 1000 + k), 0)  # obs_seed driver.hpp:77-79
        ys.append(csr_matvec(rowptr, col, val, s) + sd * noise)
    if w.noise_std is None:
        rows = np.repeat(np.arange(w.m), np.diff(rowptr))
        val = val / sd[rows]
        ys = [y / sd for y in ys]
    return (rowptr.astype(np.int32), col.astype(np.int32), val.astype(np.float64)), ys, w.sigma2


def problem(name: str, steps: int | None = None):
    """(workload, H (CsrMatrix, whitened for c3), observations, σ²) built with the product's
    host-side build_H (tomography.hpp:130-146)."""
    from . import fastkf as P
    w = CONFIGS[name]
    g = P.Grid(w.n, w.n)
    hs = [P.build_H(g, P.SourceReceiverLayout(s, r)) for s, r in layout_points(w)]
    h = P.CsrMatrix.vstack(hs) if len(hs) > 1 else hs[0]
    (rp, col, val), ys, s2 = make_inputs(w, (h.rowptr, h.col, h.val), steps)
    return w, P.CsrMatrix(h.rows, h.cols, rp, col, val), ys, s2


def kernel_spec(w: Workload):
    from . import fastkf as P
    return P.KernelSpec(family=P.MATERN, theta=w.theta, length=w.length, nu=w.nu)
