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
