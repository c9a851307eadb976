"""Sparse building blocks (mirrors markovmg/sparse.py).

Operators live in HBM as `DeviceCSR`; every product below is one engine
launch sequence with the reference's arithmetic (see csrc/sparse.cu and
csrc/spgemm.cu).  Host scipy matrices passed in are uploaded first -- that
is input ingestion, not a fallback; `make_csr` is the host-side
canonicaliser for INPUT matrices only (sparse.py:21-39).
"""

from __future__ import annotations

import numpy as np
import torch
from scipy import sparse as sp

from . import engine
from .device import DeviceCSR

STRUCTURAL_ZERO = 1e-300  # sparse.py:18


def make_csr(data, shape=None) -> sp.csr_array:
    """Canonical float64 CSR of a host INPUT (sparse.py:21-39)."""
    A = sp.csr_array(data) if sp.issparse(data) else sp.csr_array(
        np.asarray(data, dtype=np.float64), shape=shape)
    if A.dtype != np.float64:
        A = A.astype(np.float64)
    A.sum_duplicates()
    A.sort_indices()
    tiny = np.abs(A.data) < STRUCTURAL_ZERO
    if tiny.any():
        A.data[tiny] = 0.0
        A.eliminate_zeros()
    return A


def as_device(M) -> DeviceCSR:
    """DeviceCSR for a device operator or an (uploaded) host CSR input."""
    if isinstance(M, DeviceCSR):
        return M
    return DeviceCSR.from_host(make_csr(M))


def _vec(x, n=None):
    v = engine.to_device_vec(x)
    if v.dim() != 1:
        raise ValueError("expected a 1-D vector")
    if n is not None and v.shape[0] != n:
        raise ValueError(f"vector has length {v.shape[0]}, expected {n}")
    return v


def _like_input(y, x):
    return y if isinstance(x, torch.Tensor) else y.cpu().numpy()


def spmv(M, x):
    """Mx, bit-identical to scipy csr_matvec (sparse.py:81-86)."""
    A = as_device(M)
    v = _vec(x)
    if A.shape[1] != v.shape[0]:
        raise ValueError(f"dimension mismatch: matrix is {A.shape}, vector has length {v.shape[0]}")
    return _like_input(engine.spmm(A, v), x)


def spmv_transpose(M, x, Mt: DeviceCSR | None = None):
    """M^T x via the explicit sorted transpose (sparse.py:89-94)."""
    A = as_device(M)
    v = _vec(x)
    if A.shape[0] != v.shape[0]:
        raise ValueError(f"dimension mismatch: matrix is {A.shape}, vector has length {v.shape[0]}")
    T = Mt if Mt is not None else engine.transpose(A)
    return _like_input(engine.spmm(T, v), x)


def transpose(M) -> DeviceCSR:
    """Explicit transpose in canonical form (sparse.py:97-99)."""
    return engine.transpose(as_device(M))


def triple_product(Q, B, P, drop_tol: float = 0.0) -> DeviceCSR:
    """Galerkin product canon((QB)P) with scipy csr_matmat semantics (sparse.py:102-117)."""
    Qd, Bd, Pd = as_device(Q), as_device(B), as_device(P)
    if Qd.shape[1] != Bd.shape[0] or Bd.shape[1] != Pd.shape[0]:
        raise ValueError(f"dimension mismatch in triple product: {Qd.shape} x {Bd.shape} x {Pd.shape}")
    if drop_tol > 0.0:
        raise NotImplementedError("drop_tol > 0 is not on the hot path (the reference never uses it)")
    QB = engine.spgemm(Qd, Bd, order=1)
    return engine.spgemm(QB, Pd, order=0)


def adjacency_structure(M, Mt: DeviceCSR | None = None) -> DeviceCSR:
    """Pattern of M + M^T without the diagonal, unit weights (sparse.py:120-128)."""
    A = as_device(M)
    T = Mt if Mt is not None else engine.transpose(A)
    return engine.sym_pattern(A, T)


def save_matrix_market(path, M, comment: str = "") -> None:
    """Matrix Market coordinate file, 1-based, 17 significant digits (sparse.py:152-155).

    Host I/O of a result: device operators are copied down once."""
    from scipy.io import mmwrite
    from scipy import sparse as _sp
    if hasattr(M, "to_host"):
        M = M.to_host()
    mmwrite(str(path), _sp.coo_matrix(M), comment=comment, field="real", precision=17, symmetry="general")


def load_matrix_market(path):
    """Matrix Market file -> canonical CSR (sparse.py:158-160)."""
    from scipy.io import mmread
    return make_csr(mmread(str(path)))


def save_vector(path, x, comment: str = "") -> None:
    """Dense vector as an n x 1 Matrix Market array (sparse.py:163-166)."""
    from scipy.io import mmwrite
    if hasattr(x, "cpu"):
        x = x.cpu().numpy()
    mmwrite(str(path), np.asarray(x, dtype=np.float64).reshape(-1, 1), comment=comment, field="real", precision=17)


def load_vector(path) -> np.ndarray:
    """sparse.py:169-173."""
    from scipy.io import mmread
    from scipy import sparse as _sp
    arr = mmread(str(path))
    if _sp.issparse(arr):
        arr = arr.toarray()
    return np.asarray(arr, dtype=np.float64).ravel()
