"""Coarsest-level dense operators (mirrors the hot-path parts of markovmg/dense.py).

`PinvOperator` builds the explicit pseudo-inverse of the (singular) coarsest
operator on device by a one-sided Jacobi SVD with the reference's rank rule
(dense.py:118-131) and applies it as one GEMV.  The reference's `gen_sym_eig`
/ `svd` / `sym_eig` / `herm_eig_max` are LAPACK calls behind its coarsest level
and FOV tooling; here the coarsest level has its own kernels (dense.cu,
dense_large.cu, band.cu) and the FOV analysis its own (fov.py / fov.cu).
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine
from .device import DeviceCSR


class PinvOperator:
    """A^+ for a fixed square A, applied to many vectors (dense.py:118-131)."""

    def __init__(self, A, rank_tol: float = 1e-12):
        if isinstance(A, DeviceCSR):
            n = A.shape[0]
            if A.shape[0] != A.shape[1]:
                raise ValueError("square operator expected")
            D = engine.csr_to_dense(A)
        else:
            M = torch.as_tensor(np.asarray(A, dtype=np.float64))
            if M.dim() != 2 or M.shape[0] != M.shape[1]:
                raise ValueError(f"expected a square matrix, got shape {tuple(M.shape)}")
            n = M.shape[0]
            D = engine.to_device_vec(M.T.contiguous().numpy())  # column-major upload
        self.n = n
        self.Z = engine.dense_pinv(D, n, rank_tol)  # row-major n x n on device
        self.shape = (n, n)

    def apply(self, b):
        from .solver import _gemv_rowmajor
        return _gemv_rowmajor(self.Z, b)
