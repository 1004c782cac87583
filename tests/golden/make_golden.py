"""Generates tests/golden/golden.npz with an independent numpy/scipy restatement.

Nothing here uses the oracle or the product library: kernel values come from
scipy.special.kv, Γx from the dense kernel matrix (oracles.hpp:35-44), the GHEP spectrum
from a dense eigensolve of Γ^½AΓ^½ (oracles.hpp:61-73), and the filter means from a dense
Kalman filter (dense_filter.hpp:41-62).  H for the desk problems is built by a plain
Python transcription of trace_ray (tomography.hpp:29-86), kept below.

Run:  python tests/golden/make_golden.py   (regenerates golden.npz, ≈ 10 s)
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.helpers import dense_ghep, dense_kf, kernel_fn, kernel_matrix, plume_field  # noqa: E402
from paper_1405_2276_b200 import workloads as W  # noqa: E402


def trace_ray_py(nx, ny, lx, ly, src, rec):
    """tomography.hpp:29-86 in plain Python floats (IEEE double, same operation order)."""
    dx_, dy_ = rec[0] - src[0], rec[1] - src[1]
    ln = math.sqrt(dx_ * dx_ + dy_ * dy_)
    ts = [0.0, 1.0]
    gdx, gdy = lx / nx, ly / ny
    if dx_ != 0.0:
        for i in range(1, nx):
            t = (i * gdx - src[0]) / dx_
            if 0.0 < t < 1.0:
                ts.append(t)
    if dy_ != 0.0:
        for j in range(1, ny):
            t = (j * gdy - src[1]) / dy_
            if 0.0 < t < 1.0:
                ts.append(t)
    ts.sort()
    segs = []
    tp = ts[0]
    for t in ts[1:]:
        if t - tp <= 1e-12:
            continue
        h = 0.5 * (tp + t)
        mx, my = src[0] + h * dx_, src[1] + h * dy_
        ix = min(max(int(math.floor(mx / gdx)), 0), nx - 1)
        iy = min(max(int(math.floor(my / gdy)), 0), ny - 1)
        cell = ix * ny + iy
        sl = (t - tp) * ln
        if segs and segs[-1][0] == cell:
            segs[-1][1] += sl
        else:
            segs.append([cell, sl])
        tp = t
    return segs


def build_H_py(nx, ny, n_sou, n_rec):
    src = [(0.0, (i + 0.5) * 1.0 / n_sou) for i in range(n_sou)]
    rec = [(1.0, (j + 0.5) * 1.0 / n_rec) for j in range(n_rec)]
    H = np.zeros((n_sou * n_rec, nx * ny))
    row = 0
    for s in src:
        for r in rec:
            for cell, ln in trace_ray_py(nx, ny, 1.0, 1.0, s, r):
                H[row, cell] += ln
            row += 1
    return H


def main():
    from scipy.special import gamma as G, kv
    out = {}
    # kernel values: Matérn ν ∈ {½, 3/2, 5/2} and powered-exponential (kernel.hpp:51-63)
    r = np.array([0.0, 0.01, 0.05, 0.1, 0.37, 1.0, 2.5])
    for nu in (0.5, 1.5, 2.5):
        a = math.sqrt(2 * nu) * r / 0.15
        with np.errstate(invalid="ignore", divide="ignore"):
            v = 2 ** (1 - nu) / G(nu) * a ** nu * kv(nu, a)
        out[f"matern_nu{nu}"] = np.where(r == 0, 1.0, v)
    out["kernel_r"] = r
    out["powexp"] = 2.5 * np.exp(-np.sqrt(r / 0.4))
    # dense Γx on the reference's FFT-vs-dense grids (test_kernel_covariance.cpp:100-109)
    exp_kernel = dict(family=0, theta=1e-4, length=0.2, power=0.5)
    for nx, ny, lx, ly in [(20, 20, 1.0, 1.0), (13, 7, 2.0, 1.0)]:
        K = kernel_matrix(nx, ny, kernel_fn(**exp_kernel), lx, ly)
        x = W.rng_normals(nx * ny, 11, 0)
        out[f"gx_{nx}x{ny}_x"] = x
        out[f"gx_{nx}x{ny}_y"] = K @ x
    # desk GHEP spectrum (test_lowrank.cpp:117-144): 20×20, 4×6 rays, σ² = 2e-4
    H = build_H_py(20, 20, 4, 6)
    out["H_20x20_4x6"] = H
    gam = kernel_matrix(20, 20, kernel_fn(**exp_kernel))
    lam, _ = dense_ghep(H.T @ H / 2e-4, gam)
    out["ghep_lambda_20x20"] = lam[:24]
    # dense KF means (test_filters.cpp:162-191): 12×12, 3×8 rays, 10 steps, plume obs
    H12 = build_H_py(12, 12, 3, 8)
    out["H_12x12_3x8"] = H12
    ys = []
    for k in range(1, 11):
        s = plume_field(12, 12, 3.0 * k)
        ys.append(H12 @ s + math.sqrt(2e-4) * W.rng_normals(24, W.derive_seed(77, k), 0))
    out["kf12_obs"] = np.stack(ys)
    ref = dense_kf(kernel_matrix(12, 12, kernel_fn(**exp_kernel)), H12, ys, 2e-4)
    out["kf12_means"] = np.stack([m for m, _ in ref])
    out["kf12_vars"] = np.stack([np.diag(c) for _, c in ref])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
