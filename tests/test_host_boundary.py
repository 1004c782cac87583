"""CPU checks of the product boundary: libfastkf_b200.so loads and exports every symbol
include/fastkf_b200.h declares; host-side setup (build_H, trace_ray, kernel_eval,
next_smooth, the GHEP's small eigensolver) agrees bit-for-bit / to rounding with the oracle;
the replica aggregation used by bench.py works over a 2-process gloo group."""
import os
import re

import numpy as np
import pytest

import paper_1405_2276_b200 as P
from oracle import oracle as O
from paper_1405_2276_b200 import workloads as W
from paper_1405_2276_b200._native import LIB_PATH, SIGNATURES, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fastkf_b200.h")).read()
    declared = set(re.findall(r"\b(fkb_\w+)\s*\(", hdr))
    assert len(declared) > 40
    L = lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared <= set(SIGNATURES), declared - set(SIGNATURES)
    assert os.path.exists(LIB_PATH)


def test_library_has_sm100a_code():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kernel_eval_and_next_smooth_match_oracle():
    for nu in (0.5, 1.5, 2.5):
        for r in (0.0, 0.013, 0.2, 0.9):
            assert P.kernel_eval(P.KernelSpec(P.MATERN, 1.0, 0.15, nu=nu), r) == \
                O.kernel_eval(O.MATERN, 1.0, 0.15, r, nu=nu)
    for n in range(1, 300, 7):
        assert P.next_smooth(n) == O.next_smooth(n)
    with pytest.raises(ValueError):
        P.kernel_eval(P.KernelSpec(P.POWERED_EXPONENTIAL, -1.0, 0.2), 0.1)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c4"])
def test_build_H_bit_identical_to_oracle(name):
    w = W.CONFIGS[name]
    for s, r in W.layout_points(w):
        h = P.build_H(P.Grid(w.n, w.n), P.SourceReceiverLayout(s, r))
        rp, col, val = O.build_H(w.n, w.n, s, r).arrays()
        assert np.array_equal(h.rowptr, rp) and np.array_equal(h.col, col) and np.array_equal(h.val, val)
    expect_nnz = {"c0": 19776, "c1": 164480, "c2": 657920, "c4": 2697728}[name]
    assert W.problem(name, 1)[1].nnz == expect_nnz


def test_trace_ray_product_kats():
    cells, lens = P.trace_ray(P.Grid(10, 5), (0.0, 0.5), (1.0, 0.5))
    assert len(cells) == 10 and np.allclose(lens, 0.1, rtol=1e-12)
    with pytest.raises(ValueError):
        P.trace_ray(P.Grid(4, 4), (0.5, 0.5), (0.5, 0.5))
    with pytest.raises(ValueError):
        P.build_H(P.Grid(4, 4), P.SourceReceiverLayout(np.array([[-0.5, 0.5]]), np.array([[1.0, 0.5]])))


@pytest.mark.parametrize("n", [1, 2, 7, 64, 277])
def test_small_symmetric_eigensolver(n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    A = A + A.T
    w, Z = P.sym_eig(A)
    assert np.max(np.abs(w - np.linalg.eigvalsh(A))) < 1e-12 * max(1.0, np.abs(w).max())
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) < 1e-12 * n
    assert np.linalg.norm(A @ Z - Z * w) < 1e-12 * n * max(1.0, np.abs(w).max())


def test_rank_deficient_gram_eigs():
    """Null directions of a rank-deficient Gram sit at rounding level (the drop rule's gap)."""
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((200, 10)) @ rng.standard_normal((10, 14))
    w, _ = P.sym_eig(Y.T @ Y)
    assert np.sum(w > 1e-13 * w.max()) == 10


def test_workload_inputs_deterministic():
    a = W.problem("c0", 2)
    b = W.problem("c0", 2)
    assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))
    assert W.CONFIGS["c2"].ghep_sizes() == (300, 20) and W.CONFIGS["c0"].m == 256 and W.CONFIGS["c2"].m == 2048


def _replica_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = 10.0 + 5.0 * rank
    out[rank] = bench.replica_throughput(local_ms, steps=20, world=world, device="cpu")
    dist.destroy_process_group()


def test_replica_aggregation_gloo():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_replica_worker, args=(2, port, out), nprocs=2, join=True)
    # max over ranks (15 ms) → 2 replicas × 20 steps / 15 ms
    assert out[0] == pytest.approx(2 * 20 / 0.015) and out[1] == out[0]
