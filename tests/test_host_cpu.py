"""CPU-only checks: input generators, the C ABI surface, host-side config logic."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, csr_from


def _same(A, B):
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr)
            and np.array_equal(A.indices, B.indices) and np.array_equal(A.data, B.data))


@pytest.mark.parametrize("name,side", [("pipe_cfg0_tandem64", 64), ("pipe_tandem32_k16_r30", 32)])
def test_tandem_generator_bit_exact(golden, name, side):
    from paper_1402_4005_b200 import chains
    p = chains.tandem_queue(side)
    assert _same(p.B, csr_from(golden(name), "B"))
    q = chains.tandem_queue(side, validate=False)
    assert _same(q.B, p.B)
    assert np.array_equal(p.geometry, golden(name)["geometry"])


@pytest.mark.parametrize("name,side", [("pipe_uniform33", 33), ("pipe_uniform63", 63)])
def test_uniform_generator_bit_exact(golden, name, side):
    from paper_1402_4005_b200 import chains
    p = chains.uniform_2d(side)
    assert _same(p.B, csr_from(golden(name), "B"))
    assert np.array_equal(p.geometry, golden(name)["geometry"])


def test_birth_death_and_petri_generators_bit_exact(golden):
    from paper_1402_4005_b200 import chains
    assert _same(chains.birth_death(257).B, csr_from(golden("pipe_bd257_normal"), "B"))
    p = chains.petri_reachability(chains.molloy_net(10))
    assert p.n == 506
    assert _same(p.B, csr_from(golden("pipe_petri10_normal"), "B"))


def test_planar_generator_matches_reference_edges(golden):
    """Qhull vs the reference's Bowyer-Watson: identical chain at n = 1024
    except possibly convex-hull edges the reference's super-triangle misses."""
    from paper_1402_4005_b200 import chains
    p = chains.random_planar(1024, seed=1)
    ref = csr_from(golden("pipe_planar1024_k12"), "B")
    assert np.array_equal(p.geometry, golden("pipe_planar1024_k12")["geometry"])
    mine = set(zip(*p.B.nonzero()))
    theirs = set(zip(*ref.nonzero()))
    assert len(theirs - mine) == 0
    assert len(mine - theirs) <= 4  # <= 1 hull edge, both directions


def test_header_symbols_exported():
    """Every entry point include/bamg_sm100.h declares is exported by the built library."""
    from paper_1402_4005_b200 import _lib
    text = (ROOT / "include" / "bamg_sm100.h").read_text()
    names = set(re.findall(r"\b(bamg_[a-z0-9_]+)\s*\(", text))
    lib = _lib.load_library(require_gpu=False)
    assert lib.missing_symbols == []
    import ctypes
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in sorted(names):
        assert hasattr(raw, name), name
    assert names <= set(_lib.exported_symbols()), names - set(_lib.exported_symbols())


def test_no_gpu_raises_loudly():
    import torch
    from paper_1402_4005_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.BamgUnavailable):
        _lib.lib()


def test_config_validation_mirrors_reference():
    from paper_1402_4005_b200 import (CoarseningConfig, GmresConfig, InterpConfig, SetupConfig,
                                      SmootherConfig, default_setup_config)
    with pytest.raises(ValueError):
        SmootherConfig(omega=0.0)
    with pytest.raises(ValueError):
        InterpConfig(search_radius=3)
    with pytest.raises(ValueError):
        CoarseningConfig(mode="bogus")
    with pytest.raises(ValueError):
        SetupConfig(n_tests=1)
    with pytest.raises(ValueError):
        GmresConfig(rtol=0.0)
    cfg = default_setup_config("tandem", seed=0, n_tests=16)
    assert cfg.interp.caliber == 4 and cfg.coarsening.mode == "geometric2d" and cfg.n_tests == 16
