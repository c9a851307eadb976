"""The reference's acceptance criteria 6-8 (pkg/tests/test_acceptance.py:150-243),
restated against the drop-in: the same problems, seeds, tolerances and checks,
written here (the reference tree is not on the GPU box).

 6  structural invariants: 1^T B_l = 0 on every level (<= 1e-12 of the
    level's scale), 1^T Q_l = 1^T (<= 1e-13), P_l is the identity on C points;
 7  oracle equivalence at n <= 120 with two setup cycles: sigma_1 <= 1e-8,
    x within 1e-6 (l1) of the dense SVD null vector, coarsest triplets under
    identity masses equal to the dense singular values (<= 1e-9);
 8  the V-cycle is linear (<= 1e-12) and, with two levels, equals the
    two-level propagator I - C B = S^nu2 (I - P B_c^+ Q B) S^nu1 (<= 1e-10).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SEED = 1
RTOL = 1e-7


def _solve(problem, cycles, max_iters=100):
    from paper_1402_4005_b200 import GmresConfig, VCycleOperator, default_setup_config, gmres, run_setup
    cfg = default_setup_config(problem.family, cycles=cycles, seed=SEED)
    setup = run_setup(problem, cfg)
    op = VCycleOperator(setup.hierarchy, cfg.smoother)
    rep = gmres(problem.B, np.zeros(problem.n), setup.x0, GmresConfig(restart=None, max_iters=max_iters, rtol=RTOL),
                op)
    return rep, setup.hierarchy


@pytest.mark.parametrize("family,n", [("birth-death", 1025), ("birth-death", 4097), ("uniform2d", 1089),
                                      ("uniform2d", 4225), ("tandem", 1089), ("planar", 1024), ("planar", 4096)])
def test_criterion_6_structural_invariants(family, n):
    from paper_1402_4005_b200 import build_problem
    problem = build_problem(family, n=n, seed=SEED)
    rep, hierarchy = _solve(problem, 1)
    assert rep.converged
    for lev in hierarchy.levels:
        B = lev.B
        scale = np.abs(B.data).max() if B.nnz else 1.0
        colsum = np.abs(np.asarray(B.sum(axis=0))).max()
        assert colsum <= 1e-12 * max(scale, 1.0), (lev.index, colsum)
        if lev.dQ is not None:
            qdev = np.abs(np.asarray(lev.Q.sum(axis=0)).ravel() - 1.0).max()
            assert qdev <= 1e-13, (lev.index, qdev)
            Pd = lev.P.toarray()
            coarse = np.asarray(lev.split.coarse)
            eye = np.zeros((coarse.size, coarse.size))
            eye[np.arange(coarse.size), np.arange(coarse.size)] = 1.0
            assert np.array_equal(Pd[coarse], eye)


def test_criterion_7_oracle_equivalence():
    from paper_1402_4005_b200 import (GmresConfig, build_problem, coarsest_triplets, default_setup_config,
                                      run_setup, solve_steady_state)
    from scipy import sparse as sp
    for family, kw in (("birth-death", dict(n=120)), ("uniform2d", dict(n=100)), ("tandem", dict(n=100)),
                       ("planar", dict(n=100, seed=SEED)), ("petri", dict(tokens=4))):
        problem = build_problem(family, **kw)
        cfg = default_setup_config(family, cycles=2, seed=SEED)
        setup = run_setup(problem, cfg)
        assert setup.triplets.sigmas[0] <= 1e-8, family
        rep = solve_steady_state(problem, cfg, GmresConfig(max_iters=300, rtol=1e-10))
        _, _, Vt = np.linalg.svd(problem.B.toarray())
        oracle = Vt[-1]
        if oracle[np.argmax(np.abs(oracle))] < 0:
            oracle = -oracle
        oracle /= oracle.sum()
        assert rep.converged and np.abs(rep.x - oracle).sum() <= 1e-6, family
    problem = build_problem("tandem", n=100)
    eye = sp.identity(100, format="csr")
    trips = coarsest_triplets(problem.B, eye, eye, 8)
    _, s, _ = np.linalg.svd(problem.B.toarray())
    assert np.abs(trips.sigmas - s[::-1][:8]).max() <= 1e-9


def test_criterion_8_linearity_and_propagator():
    from paper_1402_4005_b200 import (VCycleOperator, build_problem, default_setup_config, degenerate_rows,
                                      run_setup)
    problem = build_problem("uniform2d", n=1089, seed=SEED)
    _, hierarchy = _solve(problem, 1)
    cfg = default_setup_config("uniform2d", cycles=1, seed=SEED)
    op = VCycleOperator(hierarchy, cfg.smoother)
    rng = np.random.default_rng(3)
    b1, b2 = rng.standard_normal((2, 1089))
    def ap(v):
        out = op.apply(v)
        return out.cpu().numpy() if hasattr(out, "cpu") else np.asarray(out)
    lhs = ap(1.3 * b1 - 0.7 * b2)
    rhs = 1.3 * ap(b1) - 0.7 * ap(b2)
    assert np.abs(lhs - rhs).max() / max(np.abs(lhs).max(), 1.0) <= 1e-12
    problem = build_problem("birth-death", n=32)
    cfg2 = default_setup_config("birth-death", cycles=1, seed=SEED)
    cfg2 = dataclasses.replace(cfg2, coarsening=dataclasses.replace(cfg2.coarsening, max_levels=2))
    setup = run_setup(problem, cfg2)
    lev = setup.hierarchy.finest
    op2 = VCycleOperator(setup.hierarchy, cfg2.smoother)
    Bd = problem.B.toarray()
    d = np.asarray(lev.diag)
    skip = degenerate_rows(problem.B, d)
    skip = skip.cpu().numpy().astype(bool) if hasattr(skip, "cpu") else np.asarray(skip, dtype=bool)
    scale = np.where(skip, 0.0, cfg2.smoother.omega / d)
    S = np.eye(32) - np.diag(scale) @ Bd
    Bc = (lev.Q @ problem.B @ lev.P).toarray()
    E = (np.linalg.matrix_power(S, cfg2.smoother.sweeps_post)
         @ (np.eye(32) - lev.P.toarray() @ np.linalg.pinv(Bc, rcond=1e-12) @ lev.Q.toarray() @ Bd)
         @ np.linalg.matrix_power(S, cfg2.smoother.sweeps_pre))
    Cd = op2.as_dense()
    Cd = Cd.cpu().numpy() if hasattr(Cd, "cpu") else np.asarray(Cd)
    assert np.abs(E - (np.eye(32) - Cd @ Bd)).max() <= 1e-10
