"""Experiment directories for the reference-style driver (tools/fkb_run.cpp), mirroring
cmd_simulate (driver.hpp:130-153): truth_stepNNN.fkf (FKF1, k = 0..n), observations.csv
("step,measurement,value", driver.hpp:91-98), plus the run parameters that the reference
keeps in config.json (experiment.txt, key value per line) and the ray layout (layout.csv:
block,role,x,y).  Per-ray noise (c3) is written as ray_std.csv and whitened by the driver
(SURVEY.md App. A.3).  Input generation only."""
from __future__ import annotations

import os

import numpy as np

from . import fastkf as P
from . import workloads as W


def simulate(out_dir: str, config: str, steps: int | None = None) -> str:
    w = W.CONFIGS[config]
    steps = w.steps if steps is None else steps
    os.makedirs(out_dir, exist_ok=True)
    g = P.Grid(w.n, w.n)
    blocks = W.layout_points(w)
    hs = [P.build_H(g, P.SourceReceiverLayout(s, r)) for s, r in blocks]
    h = P.CsrMatrix.vstack(hs) if len(hs) > 1 else hs[0]
    truths = W.truth_fields(w)[:steps]
    P.write_field(os.path.join(out_dir, "truth_step000.fkf"), w.n, w.n, np.zeros(w.N))
    for k, t in enumerate(truths, start=1):
        P.write_field(os.path.join(out_dir, f"truth_step{k:03d}.fkf"), w.n, w.n, t)
    # raw (unwhitened) observations, as simulate_observations (tomography.hpp:198-211)
    sd = W.per_ray_std(w) if w.noise_std is None else np.full(w.m, w.noise_std)
    with open(os.path.join(out_dir, "observations.csv"), "w") as f:
        f.write("step,measurement,value\n")
        for k, t in enumerate(truths, start=1):
            y = W.csr_matvec(h.rowptr, h.col, h.val, t) + sd * W.rng_normals(w.m, W.derive_seed(w.seed, 1000 + k), 0)
            f.writelines(f"{k},{i},{v!r}\n" for i, v in enumerate(y.tolist()))
    if w.noise_std is None:
        np.savetxt(os.path.join(out_dir, "ray_std.csv"), sd, fmt="%.17g")
    with open(os.path.join(out_dir, "layout.csv"), "w") as f:
        f.write("block,role,x,y\n")
        for b, (src, rec) in enumerate(blocks):
            f.writelines(f"{b},src,{x!r},{y!r}\n" for x, y in src.tolist())
            f.writelines(f"{b},rec,{x!r},{y!r}\n" for x, y in rec.tolist())
    k, p = w.ghep_sizes()
    with open(os.path.join(out_dir, "experiment.txt"), "w") as f:
        for key, val in (("nx", w.n), ("ny", w.n), ("family", 1), ("theta", w.theta), ("length", w.length),
                         ("nu", w.nu), ("sigma2", w.sigma2), ("rank", k), ("oversampling", p), ("seed", w.seed),
                         ("n_steps", steps)):
            f.write(f"{key} {val!r}\n")
    return out_dir
