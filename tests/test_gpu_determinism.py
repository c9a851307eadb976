"""Run-to-run bit identity and the hierarchy export.

* The whole path is deterministic: every reduction uses a fixed partial-sum
  tree (no floating-point atomics), the SpGEMM keeps scipy's order, and the
  parallel fits write fixed slots.  Two setups of BASELINE cfg1 (1,046,529
  states) on the same inputs give bit-identical hierarchies, x0 and x.
* export_hierarchy (bootstrap.py:447-469) writes the reference's files:
  B_l / P_l / Q_l Matrix Market, splitting_l.json, hierarchy.json.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _snapshot(setup, x):
    out = []
    for lev in setup.hierarchy.levels:
        for M in (lev.dB, lev.dM, lev.dN, lev.dP, lev.dQ):
            if M is None:
                continue
            out += [M.rowptr.clone(), M.col.clone(), M.val.clone()]
        if lev.split is not None:
            out.append(torch.as_tensor(np.asarray(lev.split.coarse)))
    out += [setup.dx0.clone(), setup.triplets.dsigmas.clone(), x.clone()]
    return out


def test_cfg1_twice_bit_identical():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import bigparity

    import paper_1402_4005_b200 as pb
    snaps = []
    for _ in range(2):
        prob, dB, cfg, setup = bigparity.run_config("cfg1")
        vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
        zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
        rep = pb.gmres(dB, zero, setup.dx0, pb.GmresConfig(rtol=1e-8), vop, to_host=False)
        snaps.append(_snapshot(setup, rep.x_device))
        del setup, vop, rep
    assert len(snaps[0]) == len(snaps[1])
    for a, b in zip(*snaps):
        assert torch.equal(a.cpu(), b.cpu())


def test_export_hierarchy_matches_reference_layout(tmp_path, golden):
    from conftest import csr_from
    from paper_1402_4005_b200 import export_hierarchy, run_setup
    from paper_1402_4005_b200.sparse import load_matrix_market
    from test_gpu_pipeline import _problem, _setup_cfg
    g = golden("pipe_uniform63")
    prob = _problem(g)
    cfg = _setup_cfg(g)
    setup = run_setup(prob, cfg, draws=(g["init_right_draw"], g["init_left_draw"]))
    export_hierarchy(setup.hierarchy, tmp_path)
    man = json.loads((tmp_path / "hierarchy.json").read_text())
    assert man["depth"] == int(g["n_levels"]) and len(man["levels"]) == man["depth"]
    for li, entry in enumerate(man["levels"]):
        ref_B = csr_from(g, f"L{li}_B")
        B = load_matrix_market(tmp_path / f"B_{li}.mtx")
        assert entry["n"] == ref_B.shape[0] and entry["nnz"] == ref_B.nnz
        assert np.array_equal(B.indptr, ref_B.indptr) and np.array_equal(B.indices, ref_B.indices)
        assert np.abs(B.data - ref_B.data).max() <= 1e-9 * np.abs(ref_B.data).max()
        if li < man["depth"] - 1:
            for key in ("P", "Q"):
                M = load_matrix_market(tmp_path / f"{key}_{li}.mtx")
                R = csr_from(g, f"L{li}_{key}")
                assert np.array_equal(M.indptr, R.indptr) and np.array_equal(M.indices, R.indices)
            sp_doc = json.loads((tmp_path / entry["splitting"]).read_text())
            assert sp_doc["coarse"] == g[f"L{li}_coarse"].tolist() and entry["n_coarse"] == len(sp_doc["coarse"])
