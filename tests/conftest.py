"""Shared pytest plumbing: the `gpu` marker and golden-fixture loaders."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


PIPE_CASES = ["pipe_cfg0_tandem64", "pipe_tandem32_k16_r30", "pipe_uniform33",
              "pipe_uniform63", "pipe_planar1024_k12", "pipe_bd257_normal",
              "pipe_petri10_normal", "pipe2_tandem33_bamg2", "pipe2_uniform33_bamg2"]


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def csr_from(g, prefix):
    from scipy import sparse as sp
    shape = tuple(int(v) for v in g[prefix + "_shape"])
    return sp.csr_array((g[prefix + "_data"], g[prefix + "_indices"].astype(np.int32),
                         g[prefix + "_indptr"].astype(np.int32)), shape=shape)


def oracle_cfg(g):
    """Rebuild the oracle config dict from a pipeline fixture."""
    ci = [int(v) for v in g["cfg_ints"]]
    cf = [float(v) for v in g["cfg_floats"]]
    return {
        "k": ci[0], "cycles": ci[1], "omega": cf[0], "nu_pre": ci[3], "nu_post": ci[4],
        "interp": {"caliber": ci[5], "radius": ci[6], "tol": cf[1],
                   "constrain_q": bool(ci[7]), "nonneg": bool(ci[8])},
        "stop": ci[9], "max_levels": ci[11], "mode": str(g["cfg_mode"]),
        "cr_sweeps": ci[10], "cr_threshold": cf[2], "cr_omega": cf[3], "seed": ci[12],
    }


def gmres_args(g):
    restart, max_iters, rtol = [float(v) for v in g["gmres"]]
    return (None if restart < 0 else int(restart)), int(max_iters), rtol


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get
