"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by running the reference (`make_golden.py`); the
oracle calls the same numpy/scipy primitives, so on a host with the same
library stack every array must agree bit for bit.  Patterns (splits, CSR
structure) are compared exactly on any host; values to 1e-12 relative where
BLAS kernels differ between hosts.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import PIPE_CASES, csr_from, gmres_args, oracle_cfg
from oracle import bamg_oracle as orc


def same_pattern(A, B):
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr)
            and np.array_equal(A.indices, B.indices))


def close(a, b, rel=1e-12):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.abs(b).max(initial=0.0), 1e-300)
    return np.abs(a - b).max(initial=0.0) <= rel * scale


@pytest.mark.parametrize("name", PIPE_CASES)
def test_pipeline_matches_reference(name, golden):
    g = golden(name)
    B = csr_from(g, "B")
    cfg = oracle_cfg(g)
    restart, max_iters, rtol = gmres_args(g)
    geometry = g.get("geometry")
    trace = {}
    levels, T, x0, its, hist, conv, x = orc.solve(
        B, cfg, geometry, g["init_right_draw"], g["init_left_draw"], restart, rtol,
        max_iters, trace)
    assert len(levels) == int(g["n_levels"])
    assert len(trace.get("splits", [])) == int(g["n_splits"])
    for i, c in enumerate(trace.get("splits", [])):
        assert np.array_equal(c, g[f"split{i}"]), f"split {i}"
    for li, L in enumerate(levels):
        for key, M in (("B", L.B), ("M", L.M), ("N", L.N), ("P", L.P), ("Q", L.Q)):
            if M is None:
                continue
            ref = csr_from(g, f"L{li}_{key}")
            assert same_pattern(M, ref), f"level {li} {key} pattern"
            assert close(M.data, ref.data), f"level {li} {key} values"
    for i, w in enumerate(trace.get("vw", [])):
        assert close(w, g[f"vw{i}"])
    assert close(x0, g["x0"], 1e-10)
    assert its == int(g["iterations"])
    assert np.abs(x - g["x"]).sum() <= 1e-10
    assert close(hist, g["history"], 1e-6)


def test_sparse_kernels_match_reference(golden):
    g = golden("kernels")
    A = csr_from(g, "A")
    assert np.array_equal(orc.mv(A, g["x"]), g["Ax"])
    assert np.array_equal(orc.mtv(A, g["x"]), g["ATx"])
    AT = orc.explicit_transpose(A)
    ref = csr_from(g, "AT")
    assert same_pattern(AT, ref) and np.array_equal(AT.data, ref.data)
    assert same_pattern(orc.sym_pattern(A), csr_from(g, "adjA"))
    C = orc.galerkin(csr_from(g, "tpQ"), csr_from(g, "tpB"), csr_from(g, "tpP"))
    ref = csr_from(g, "tpC")
    assert same_pattern(C, ref) and np.array_equal(C.data, ref.data)


def test_jacobi_matches_reference(golden):
    g = golden("kernels")
    B = csr_from(g, "jacB")
    d = B.diagonal()
    sk = orc.skip_rows(B, d)
    skt = orc.skip_rows(B, d, along_columns=True)
    assert np.array_equal(sk, g["jac_skip"]) and np.array_equal(skt, g["jac_skip_t"])
    assert np.array_equal(orc.sweep(B, g["jac_x"], g["jac_b"], 0.7, d, sk), g["jac_out"])
    assert np.array_equal(orc.sweep(B, g["jac_x"], g["jac_b"], 0.7, d, skt, True),
                          g["jac_out_t"])


def test_fit_row_matches_reference(golden):
    g = golden("kernels")
    for i in range(int(g["fit_n"])):
        r, m, cal, con, nn = [int(v) for v in g[f"fit{i}_meta"]]
        sel, coef, val = orc.greedy_fit(g[f"fit{i}_y"], g[f"fit{i}_C"], g[f"fit{i}_w"], cal,
                                        1e-3, bool(con), float(g[f"fit{i}_ridge"]), bool(nn))
        assert np.array_equal(sel, g[f"fit{i}_sel"]), i
        assert close(coef, g[f"fit{i}_coef"]), i
        assert close([val], [g[f"fit{i}_val"]]), i


def test_cr_split_matches_reference(golden):
    g = golden("kernels")
    s = orc.cr_split(csr_from(g, "crB"), 5, 0.78, 0.7, np.random.SeedSequence(11))
    assert np.array_equal(s.coarse, g["cr_coarse"])


def test_coarsest_triplets_match_reference(golden):
    from scipy import sparse as sp
    g = golden("kernels")
    B = csr_from(g, "ctB")
    M = sp.csr_array(np.diag(g["ct_M"]))
    N = sp.csr_array(np.diag(g["ct_N"]))
    T = orc.exact_triplets(B, M, N, 6)
    assert close(T.sig, g["ct_sigmas"], 1e-9)
    # singular vectors are defined up to a joint sign
    for j in range(T.r):
        s = np.sign(T.right[j] @ g["ct_right"][j])
        assert close(s * T.right[j], g["ct_right"][j], 1e-8)
        assert close(s * T.left[j], g["ct_left"][j], 1e-8)


def test_pinv_matches_reference(golden):
    g = golden("kernels")
    B = csr_from(g, "ctB").toarray()
    assert close(orc.pinv_apply(B, g["pinv_b"]), g["pinv_out"], 1e-12)
