"""GPU parity of the greedy weighted ridge LS fit (interp.py:129-238).

Each of the reference's 64 seeded fit_row cases (tests/golden/kernels.npz:
random r, m, caliber, constrain / nonnegative flags, ridge in {0, 0.01, 0.3},
an infinite-weight slot every fourth case) is posed as a tiny level -- one
fine point whose candidates are the m coarse points -- and fitted by the
engine on both paths: the thread-per-point normal-equation path (production)
and the warp Householder-QR path (forced with BAMG_FIT_WARP=1; also what the
ridge = 0 cases take).  Selected candidates must match exactly (order
included), coefficients to 1e-10 relative.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pose(y, C, w):
    """(adj, crank, X, w) for a level with point 0 fine and points 1..m coarse."""
    from paper_1402_4005_b200.device import DeviceCSR
    r, m = C.shape
    n = m + 1
    rp = np.concatenate([[0, m], m + np.arange(1, m + 1)]).astype(np.int32)
    ci = np.concatenate([np.arange(1, m + 1), np.zeros(m)]).astype(np.int32)
    adj = DeviceCSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                    torch.ones(2 * m, dtype=torch.float64, device="cuda"), (n, n))
    crank = torch.from_numpy(np.concatenate([[-1], np.arange(m)]).astype(np.int32)).cuda()
    X = np.zeros((n, r))
    X[0] = y
    X[1:] = C.T
    return adj, crank, torch.from_numpy(X).cuda(), torch.from_numpy(np.asarray(w, dtype=np.float64)).cuda()


def _decision_margin(y, C, w, caliber, constrain, ridge, nonneg, tol=1e-3):
    """Smallest relative margin of the greedy's decisions (argmin gaps and the
    improvement-stop test), replayed with the oracle.  Cases decided by
    rounding noise (exact fits, r <= number of columns) have margin ~0: no
    independent arithmetic can reproduce LAPACK's noise, so they are not
    parity cases."""
    from oracle import bamg_oracle as orc
    fin = np.isfinite(w)
    empty = float(np.sum(w[fin] * y[fin] ** 2))
    scale = max(empty, 1e-300)
    chosen, margin, cur = [], np.inf, empty
    m = C.shape[1]
    while len(chosen) < min(caliber, m):
        totals = []
        for j in range(m):
            if j in chosen:
                continue
            cols = chosen + [j]
            sw = np.sqrt(w[fin])
            yf, Cf = y[fin], C[fin]
            if constrain and len(cols) > 1:
                _, _, tot = orc._ridge_ls(Cf[:, cols[1:]] - Cf[:, [cols[0]]], yf - Cf[:, cols[0]], sw, ridge)
            elif constrain:
                res = sw * (yf - Cf[:, cols[0]])
                tot = float(res @ res)
            else:
                _, _, tot = orc._ridge_ls(Cf[:, cols], yf, sw, ridge)
            totals.append((tot, j))
        totals.sort()
        if len(totals) > 1:
            margin = min(margin, (totals[1][0] - totals[0][0]) / scale)
        best, j = totals[0]
        if chosen:
            margin = min(margin, abs((cur - best) - tol * cur) / scale)
            if cur <= 0.0 or (cur - best) < tol * cur:
                break
        chosen.append(j)
        cur = best
        if cur <= 1e-30:
            break
    return margin


@pytest.mark.parametrize("path", ["thread", "warp"])
def test_fit_row_cases_match_reference(golden, path, monkeypatch):
    from paper_1402_4005_b200 import engine
    if path == "warp":
        monkeypatch.setenv("BAMG_FIT_WARP", "1")
    else:
        monkeypatch.delenv("BAMG_FIT_WARP", raising=False)
    g = golden("kernels")
    bad = []
    checked = 0
    for i in range(int(g["fit_n"])):
        r, m, cal, con, nn = [int(v) for v in g[f"fit{i}_meta"]]
        ridge = float(g[f"fit{i}_ridge"])
        if _decision_margin(g[f"fit{i}_y"], g[f"fit{i}_C"], g[f"fit{i}_w"], cal, bool(con), ridge,
                            bool(nn)) < 1e-9:
            continue  # decided by rounding noise in the reference
        checked += 1
        adj, crank, X, w = _pose(g[f"fit{i}_y"], g[f"fit{i}_C"], g[f"fit{i}_w"])
        cnt, col, val, status = engine.fit_rows(adj, crank, X, w, cal, 1, 1e-3, bool(con), bool(nn),
                                                ridge=ridge)
        c = int(cnt[0].item())
        sel = col[:c].cpu().numpy()
        coef = val[:c].cpu().numpy()
        ref_sel = g[f"fit{i}_sel"]
        ref_coef = g[f"fit{i}_coef"]
        scale = max(np.abs(ref_coef).max(initial=0.0), 1e-300)
        if not (np.array_equal(sel, ref_sel) and np.abs(coef - ref_coef).max(initial=0.0) <= 1e-10 * scale):
            bad.append((i, sel.tolist(), ref_sel.tolist(), coef.tolist(), ref_coef.tolist()))
    assert not bad, bad[:3]
    assert checked >= 40, checked


def test_thread_and_warp_paths_agree_on_a_level(golden, monkeypatch):
    """Both fit paths on a real level (uniform 63x63, golden initial vectors)."""
    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200 import engine
    from paper_1402_4005_b200.bootstrap import _LevelOps
    from conftest import csr_from
    g = golden("pipe_uniform63")
    B = pb.DeviceCSR.from_host(csr_from(g, "B"))
    ops = _LevelOps(B)
    split = pb.geometric_coarsen(g["geometry"], "geometric2d")
    V = torch.from_numpy(np.ascontiguousarray(g["sm0_right"].T)).cuda()
    U = torch.from_numpy(np.ascontiguousarray(g["sm0_left"].T)).cuda()
    vt = pb.singular_test_weights(B, V)
    ut = pb.singular_test_weights(B, U, transpose_side=True, infinite_slot=0, Bt=ops.Bt)
    out = {}
    for path in ("thread", "warp"):
        if path == "warp":
            monkeypatch.setenv("BAMG_FIT_WARP", "1")
        else:
            monkeypatch.delenv("BAMG_FIT_WARP", raising=False)
        res = []
        for tests, constrain in ((vt, False), (ut, True)):
            cnt, col, val, st = engine.fit_rows(ops.adj, split.dcrank, tests.dvectors, tests.dweights, 4, 1,
                                                1e-3, constrain, True)
            res.append((cnt.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy(), st))
        out[path] = res
    for (c1, k1, v1, s1), (c2, k2, v2, s2) in zip(out["thread"], out["warp"]):
        assert s1[1] == 0  # nothing deferred on this level
        assert np.array_equal(c1, c2)
        mask = np.repeat(np.arange(4)[None, :], c1.size, 0) < c1[:, None]
        assert np.array_equal(k1.reshape(-1, 4)[mask], k2.reshape(-1, 4)[mask])
        a, b = v1.reshape(-1, 4)[mask], v2.reshape(-1, 4)[mask]
        assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()
    # and the resulting P / W patterns equal the reference's
    P = engine.rows_to_csr(*[torch.from_numpy(x).cuda() for x in out["thread"][0][:3]], split.n, 4,
                           split.n_coarse).to_host()
    ref = csr_from(g, "fitP0")
    assert np.array_equal(P.indptr, ref.indptr) and np.array_equal(P.indices, ref.indices)
