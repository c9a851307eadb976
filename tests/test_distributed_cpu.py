"""Multi-process (gloo, world_size 2, CPU) tests of the row-partition host logic."""

from __future__ import annotations

import socket

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_partition_balanced():
    from paper_1402_4005_b200.distributed import RowPartition
    p = RowPartition(10, 3)
    assert p.offsets.tolist() == [0, 4, 7, 10]
    assert p.owner([0, 3, 4, 9]).tolist() == [0, 0, 1, 2]


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plans_reproduce_global_spmv(tmp_path, world):
    import torch.multiprocessing as mp
    import dist_workers
    mp.spawn(dist_workers.plan_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok = np.load(tmp_path / f"plan_{r}.npy")
        assert ok.all(), (r, ok)


@pytest.mark.parametrize("world", [2, 3])
def test_slot_partition_column_gather(tmp_path, world):
    """The multi-GPU setup splits the k triplet slots over the ranks; the column all-gather
    must rebuild the n x k block for even and uneven splits (k = 16, 12, 7)."""
    import torch.multiprocessing as mp
    import dist_workers
    mp.spawn(dist_workers.cols_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"cols_{r}.npy").all()


def test_gram_form_coefficients_equal_cgs2():
    """Host side of the two-pass Arnoldi step (distributed.py / csrc/solver.cu): with
    G = V^T V of a slightly non-orthonormal basis, c = 2 h1 - G h1 are CGS2's total
    coefficients and |w|^2 - 2 c.h1 + c^T G c is |w - V c|^2."""
    rng = np.random.default_rng(5)
    n, m = 4000, 9
    V, _ = np.linalg.qr(rng.standard_normal((n, m)))
    V = V + 1e-9 * rng.standard_normal((n, m))   # round-off-like defects
    w = rng.standard_normal(n) + V @ rng.standard_normal(m) * 5.0
    G = V.T @ V
    h1 = V.T @ w
    c = h1 + (h1 - G @ h1)
    w1 = w - V @ h1
    h2 = V.T @ w1
    assert np.allclose(c, h1 + h2, rtol=0, atol=1e-12 * np.abs(h1).max())
    eta2 = (w @ w - c @ h1) - (c @ h1 - c @ (G @ c))
    assert abs(eta2 - np.sum((w - V @ c) ** 2)) <= 1e-10 * (w @ w)
