"""The engine's own fp64 GEMM / GEMV (csrc/gemm.cu) against a torch fp64 reference.

These kernels replace the BLAS behind the reference's dense coarsest level
(dense.py:53-131 through numpy/LAPACK).  Tolerance: fp64 products with
different summation order agree to ~k * 2^-53 relative; we ask for 1e-12 of
the |A||B| scale.
"""

from __future__ import annotations

import itertools

import pytest
import torch

pytestmark = pytest.mark.gpu


def run_gemm(ta, tb, m, n, k, alpha, beta, lda_pad=0, ldb_pad=0, ldc_pad=0, seed=0):
    from paper_1402_4005_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(seed)
    ar, ac = (k, m) if ta else (m, k)
    br, bc = (n, k) if tb else (k, n)
    lda, ldb, ldc = ar + lda_pad, br + ldb_pad, m + ldc_pad
    # column-major storage: a (cols x ld) row-major tensor is an (ld x cols) column-major one
    A = torch.randn(ac, lda, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(bc, ldb, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(n, ldc, dtype=torch.float64, device="cuda", generator=g)
    Am = A[:, :ar].T  # ar x ac
    Bm = B[:, :br].T
    opA = Am.T if ta else Am
    opB = Bm.T if tb else Bm
    ref = alpha * (opA @ opB) + beta * C[:, :m].T
    C0 = C.clone()
    _lib.call("bamg_dgemm", int(ta), int(tb), m, n, k, alpha, _lib.ptr(A), lda, _lib.ptr(B), ldb, beta,
              _lib.ptr(C), ldc)
    torch.cuda.synchronize()
    got = C[:, :m].T
    scale = (opA.abs() @ opB.abs()).abs().max().item() * abs(alpha) + abs(beta) * C0.abs().max().item() + 1e-300
    err = (got - ref).abs().max().item() / scale
    # the padding rows of C stay untouched
    assert torch.equal(C[:, m:], C0[:, m:])
    return err


@pytest.mark.parametrize("ta,tb", list(itertools.product([False, True], repeat=2)))
@pytest.mark.parametrize("m,n,k", [(300, 257, 129), (1, 77, 500), (513, 1, 700), (40, 24, 5000),
                                   (2000, 28, 1900), (28, 2000, 300), (130, 140, 3), (64, 64, 0)])
def test_dgemm_matches_torch(ta, tb, m, n, k):
    err = run_gemm(ta, tb, m, n, k, alpha=-1.5, beta=0.5, lda_pad=3, ldb_pad=1, ldc_pad=5)
    assert err < 1e-13, err


def test_dgemm_beta_zero_ignores_nan_output():
    from paper_1402_4005_b200 import _lib
    m = n = k = 96
    A = torch.randn(k, m, dtype=torch.float64, device="cuda")
    B = torch.randn(n, k, dtype=torch.float64, device="cuda")
    C = torch.full((n, m), float("nan"), dtype=torch.float64, device="cuda")
    _lib.call("bamg_dgemm", 0, 0, m, n, k, 1.0, _lib.ptr(A), m, _lib.ptr(B), k, 0.0, _lib.ptr(C), m)
    ref = A.T @ B.T
    assert torch.allclose(C.T, ref, rtol=1e-13, atol=1e-12)


def test_dgemm_large_square_and_deterministic():
    err = run_gemm(False, True, 2304, 2176, 2048, alpha=1.0, beta=0.0)
    assert err < 1e-13, err
    from paper_1402_4005_b200 import _lib
    A = torch.randn(48, 6000, dtype=torch.float64, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.zeros(48, 48, dtype=torch.float64, device="cuda")
        _lib.call("bamg_dgemm", 1, 0, 48, 48, 6000, 1.0, _lib.ptr(A), 6000, _lib.ptr(A), 6000, 0.0,
                  _lib.ptr(C), 48)
        outs.append(C.clone())
    assert torch.equal(outs[0], outs[1])  # split-k reduction in fixed order
