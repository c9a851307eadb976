"""Device-resident CSR operators and vector blocks.

`DeviceCSR` keeps the three CSR arrays of one operator in HBM (int32
rowptr/col, fp64 values) as torch tensors -- torch is the allocator here, not
the compute -- and hands the engine a `bamg_csr` descriptor.  Conversion to a
host `scipy.sparse.csr_array` happens only on explicit request (lazy
attribute access on `Level`, tests, export), never inside the compute path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
from scipy import sparse as sp

from . import _lib


def device():
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


class DeviceCSR:
    __slots__ = ("rowptr", "col", "val", "shape", "_desc", "is_identity", "packed", "dict", "pslice",
                 "ptiles", "stencil")

    def __init__(self, rowptr, col, val, shape, is_identity=False):
        self.rowptr = rowptr
        self.col = col
        self.val = val
        self.shape = (int(shape[0]), int(shape[1]))
        self.is_identity = is_identity
        self._desc = None
        # packed copy for the k = 1 kernels (engine.pack_operator), else None
        self.packed = None
        self.dict = None
        self.pslice = None
        # stencil (engine.attach_stencil): the tile flags (device) and the
        # filled descriptor bamg_csr_stencil returned (the st_* fields are copied from it)
        self.ptiles = None
        self.stencil = None

    @property
    def nnz(self) -> int:
        return int(self.col.numel())

    @property
    def n(self) -> int:
        return self.shape[0]

    def desc(self):
        if self._desc is None:
            self._desc = _lib.CSR(self.shape[0], self.shape[1], self.nnz,
                                  self.rowptr.data_ptr(),
                                  self.col.data_ptr() if self.nnz else None,
                                  self.val.data_ptr() if self.nnz else None,
                                  self.packed.data_ptr() if self.packed is not None else None,
                                  self.dict.data_ptr() if self.dict is not None else None,
                                  self.pslice.data_ptr() if self.pslice is not None else None,
                                  int(self.packed.numel()) if self.packed is not None else 0)
            st = self.stencil
            if st is not None and self.ptiles is not None:
                d = self._desc
                d.ptiles = self.ptiles.data_ptr()
                d.st_w, d.st_diag, d.st_d, d.st_rd, d.st_tiles = st.st_w, st.st_diag, st.st_d, st.st_rd, st.st_tiles
                for u in range(8):
                    d.st_delta[u] = st.st_delta[u]
                    d.st_val[u] = st.st_val[u]
        return self._desc

    def ref(self):
        return C.byref(self.desc())

    @classmethod
    def from_host(cls, M, dev=None, non_blocking=False):
        """Upload a canonical scipy CSR (the caller's host input)."""
        dev = dev or device()
        M = sp.csr_array(M)
        if M.shape[0] >= 2 ** 31 or M.nnz >= 2 ** 31:
            raise ValueError("operators in scope have int32 indices")
        rp = torch.from_numpy(np.ascontiguousarray(M.indptr, dtype=np.int32))
        ci = torch.from_numpy(np.ascontiguousarray(M.indices, dtype=np.int32))
        va = torch.from_numpy(np.ascontiguousarray(M.data, dtype=np.float64))
        if non_blocking:
            rp, ci, va = rp.pin_memory(), ci.pin_memory(), va.pin_memory()
        return cls(rp.to(dev, non_blocking=non_blocking), ci.to(dev, non_blocking=non_blocking),
                   va.to(dev, non_blocking=non_blocking), M.shape)

    @classmethod
    def identity(cls, n, dev=None):
        dev = dev or device()
        rp = torch.arange(n + 1, dtype=torch.int32, device=dev)
        ci = torch.arange(n, dtype=torch.int32, device=dev)
        va = torch.ones(n, dtype=torch.float64, device=dev)
        return cls(rp, ci, va, (n, n), is_identity=True)

    def to_host(self) -> sp.csr_array:
        return sp.csr_array((self.val.cpu().numpy(), self.col.cpu().numpy(),
                             self.rowptr.cpu().numpy()), shape=self.shape)


def empty(n, k=1, dtype=torch.float64):
    shape = (n,) if k == 1 else (n, k)
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(n, k=1, dtype=torch.float64):
    shape = (n,) if k == 1 else (n, k)
    return torch.zeros(shape, dtype=dtype, device=device())


def i64ref():
    v = C.c_int64(0)
    return v, C.byref(v)
