"""Thin typed wrappers over the C ABI (include/bamg_sm100.h).

Every function here allocates its outputs with torch (HBM allocator only),
binds every argument to a local before the call (a tensor freed before the
launch is enqueued could be handed to the next allocation), and launches
exactly one engine entry point.  No arithmetic happens in Python.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .device import DeviceCSR, device

F64 = torch.float64
I32 = torch.int32
U8 = torch.uint8


def _p(t):
    return _lib.ptr(t)


def _dev():
    return device()


def _empty(shape, dtype=F64):
    return torch.empty(shape, dtype=dtype, device=_dev())


def _block(X):
    """(tensor, n, k) of an n x k interleaved block (1-D -> k = 1)."""
    if X.dim() == 1:
        return X, X.shape[0], 1
    return X, X.shape[0], X.shape[1]


def to_device_vec(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(), dtype=F64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(_dev())


# ----------------------------------------------------------------- sparse
def spmm(A: DeviceCSR, X):
    X, n, k = _block(X)
    if n != A.shape[1]:
        raise ValueError(f"dimension mismatch: matrix is {A.shape}, vector has length {n}")
    Y = _empty((A.shape[0],) if X.dim() == 1 else (A.shape[0], k))
    _lib.call("bamg_spmm", A.ref(), _p(X), _p(Y), k)
    return Y


def pack_operator(A: DeviceCSR) -> bool:
    """Attach the packed (value-indexed, 32-bit, slice-major) copy the k = 1 kernels
    stream instead of rowptr / col / val (bamg_csr_pack_plan / _fill).  True when A
    qualifies (<= 254 distinct values, |col - row| < 2^23); otherwise A is left as it is."""
    A.packed = A.dict = A.pslice = A.ptiles = A.stencil = None
    A._desc = None
    if A.shape[0] != A.shape[1] or A.nnz == 0:
        return False
    pslice = _empty((A.shape[0] + 31) // 32 + 1, I32)
    dic = _empty(512, F64)
    nd, words = C.c_int(0), C.c_int64(0)
    _lib.call("bamg_csr_pack_plan", A.ref(), _p(pslice), _p(dic), C.byref(nd), C.byref(words))
    if not nd.value:
        return False
    packed = _empty(max(words.value, 1), I32)
    _lib.call("bamg_csr_pack_fill", A.ref(), _p(pslice), _p(dic), nd.value, _p(packed))
    A.packed, A.dict, A.pslice = packed, dic, pslice
    A._desc = None
    attach_stencil(A)
    return True


def attach_stencil(A: DeviceCSR) -> bool:
    """Flag the 256-row tiles of a lattice operator whose rows all carry the interior row's
    (col - row, value) list (bamg_csr_stencil); the k = 1 packed kernels and the k-wide sweeps
    take those tiles' offsets and values from their parameter space.  False (A unchanged) for
    operators without a dominant row: meshes, Galerkin levels."""
    A.ptiles = A.stencil = None
    A._desc = None
    if os.environ.get("BAMG_NO_STENCIL") == "1" or A.shape[0] != A.shape[1] or A.nnz == 0:
        return False
    tiles = _empty((A.shape[0] + 255) // 256, U8)
    out = _lib.CSR()
    _lib.call("bamg_csr_stencil", A.ref(), _p(tiles), C.byref(out))
    if not out.ptiles:
        return False
    A.ptiles, A.stencil = tiles, out
    A._desc = None
    return True
    tiles = _empty((A.shape[0] + 255) // 256, U8)
    out = _lib.CSR()
    _lib.call("bamg_csr_pack_stencil", A.ref(), _p(tiles), C.byref(out))
    if out.ptiles:
        A.ptiles, A.stencil = tiles, out
        A._desc = None
    return True


def transpose(A: DeviceCSR) -> DeviceCSR:
    rp = _empty(A.shape[1] + 1, I32)
    ci = _empty(A.nnz, I32)
    va = _empty(A.nnz, F64)
    _lib.call("bamg_csr_transpose", A.ref(), _p(rp), _p(ci), _p(va))
    return DeviceCSR(rp, ci, va, (A.shape[1], A.shape[0]))


def sym_pattern(A: DeviceCSR, At: DeviceCSR) -> DeviceCSR:
    rp = _empty(A.shape[0] + 1, I32)
    nnz = C.c_int64(0)
    _lib.call("bamg_sym_pattern_count", A.ref(), At.ref(), _p(rp), C.byref(nnz))
    ci = _empty(max(nnz.value, 1), I32)[: nnz.value]
    _lib.call("bamg_sym_pattern_fill", A.ref(), At.ref(), _p(rp), _p(ci))
    ones = torch.ones(nnz.value, dtype=F64, device=_dev())
    return DeviceCSR(rp, ci, ones, A.shape)


def diag(A: DeviceCSR):
    d = _empty(min(A.shape))
    _lib.call("bamg_diag", A.ref(), _p(d))
    return d


def count_nonpositive(d) -> int:
    out = C.c_int64(0)
    _lib.call("bamg_count_nonpositive", _p(d), d.numel(), C.byref(out))
    return out.value


def count_empty_rows(A: DeviceCSR) -> int:
    out = C.c_int64(0)
    _lib.call("bamg_count_empty_rows", A.ref(), C.byref(out))
    return out.value


SPGEMM_STORAGE, SPGEMM_REV_A, SPGEMM_REV_B = 1, 2, 4  # bamg_spgemm_count `order` bits


def spgemm(A: DeviceCSR, B: DeviceCSR, order: int = 0) -> DeviceCSR:
    """C = A B with scipy csr_matmat semantics; `order` 0 canonical, 1 scipy
    storage order, optionally | SPGEMM_REV_A / SPGEMM_REV_B (rows walked in
    reverse: the products with an identity mass folded in)."""
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"dimension mismatch in sparse product: {A.shape} x {B.shape}")
    rp = _empty(A.shape[0] + 1, I32)
    nnz = C.c_int64(0)
    _lib.call("bamg_spgemm_count", A.ref(), B.ref(), order, _p(rp), C.byref(nnz))
    ci = _empty(max(nnz.value, 1), I32)
    va = _empty(max(nnz.value, 1), F64)
    _lib.call("bamg_spgemm_fill", A.ref(), B.ref(), order, _p(rp), _p(ci), _p(va))
    return DeviceCSR(rp, ci[: nnz.value], va[: nnz.value], (A.shape[0], B.shape[1]))


def spgemm_many(products):
    """Independent products [(A, B, order), ...] (at most 4): counts issued
    together, ONE host read for all their sizes, then the fills.  Same results
    as spgemm() on each."""
    if not 1 <= len(products) <= 4:
        raise ValueError("1..4 products per batch")
    rps, keep = [], []
    for slot, (A, B, order) in enumerate(products):
        if A.shape[1] != B.shape[0]:
            raise ValueError(f"dimension mismatch in sparse product: {A.shape} x {B.shape}")
        rp = _empty(A.shape[0] + 1, I32)
        ra, rb = A.ref(), B.ref()
        keep += [ra, rb]
        _lib.call("bamg_spgemm_count_slot", ra, rb, order, _p(rp), slot)
        rps.append(rp)
    slots = (C.c_int32 * len(products))(*range(len(products)))
    nnz = (C.c_int64 * len(products))()
    _lib.call("bamg_spgemm_count_wait", len(products), slots, nnz)
    out = []
    for slot, ((A, B, order), rp) in enumerate(zip(products, rps)):
        m = int(nnz[slot])
        ci = _empty(max(m, 1), I32)
        va = _empty(max(m, 1), F64)
        _lib.call("bamg_spgemm_fill_slot", A.ref(), B.ref(), order, _p(rp), _p(ci), _p(va), slot)
        out.append(DeviceCSR(rp, ci[:m], va[:m], (A.shape[0], B.shape[1])))
    return out


# ------------------------------------------------------------------ relax
def degenerate_rows(A: DeviceCSR, d):
    skip = _empty(A.shape[0], U8)
    _lib.call("bamg_degenerate_rows", A.ref(), _p(d), _p(skip))
    return skip


def jacobi(A: DeviceCSR, d, skip, x, b=None, b_scale=None, omega=0.7, peak=None):
    x, n, k = _block(x)
    out = torch.empty_like(x)
    _lib.call("bamg_jacobi", A.ref(), _p(d), _p(skip), _p(b), _p(b_scale), _p(x), _p(out), k,
              float(omega), _p(peak))
    return out


# ---------------------------------------------------------- block helpers
def col_norms(X):
    X, n, k = _block(X)
    out = _empty(k)
    _lib.call("bamg_col_norms", _p(X), n, k, _p(out))
    return out


def col_dots(X, Y):
    X, n, k = _block(X)
    out = _empty(k)
    _lib.call("bamg_col_dots", _p(X), _p(Y), n, k, _p(out))
    return out


def normalize_cols(X):
    """In place: X[:, c] /= ||X[:, c]|| (zero norms left alone)."""
    X, n, k = _block(X)
    nrm = col_norms(X)
    _lib.call("bamg_col_scale_div", _p(X), n, k, _p(nrm))
    return X


def col_fill(X, c, value):
    X, n, k = _block(X)
    _lib.call("bamg_col_fill", _p(X), n, k, int(c), float(value))


def gather_rows(X, idx):
    X, n, k = _block(X)
    m = idx.numel()
    Y = _empty((m,) if X.dim() == 1 else (m, k))
    _lib.call("bamg_gather_rows", _p(X), _p(idx), m, k, _p(Y))
    return Y


def permute_cols(X, perm):
    X, n, k = _block(X)
    arr = (C.c_int32 * k)(*[int(v) for v in perm])
    Y = torch.empty_like(X)
    _lib.call("bamg_permute_cols", _p(X), n, k, arr, _p(Y))
    return Y


# -------------------------------------------------------------- bootstrap
def smooth_block(A, At, M, N, d, skip, skip_t, U, V, sigma, nsweeps, omega, inhomogeneous,
                 smooth=1, refresh=1):
    n, k = V.shape
    _lib.call("bamg_smooth_block", A.ref(), At.ref(), M.ref() if M is not None else None,
              N.ref() if N is not None else None, _p(d), _p(skip), _p(skip_t), _p(U), _p(V),
              _p(sigma), k, int(nsweeps), float(omega), int(inhomogeneous), int(smooth), int(refresh))


def refresh_sigmas(A, M, N, U, V, sigma, flip=True):
    n, k = V.shape
    _lib.call("bamg_refresh_sigmas", A.ref(), M.ref() if M is not None else None,
              N.ref() if N is not None else None, _p(U), _p(V), _p(U) if flip else None,
              _p(sigma), k)


# ------------------------------------------------------------------ interp
def test_weights(A, X, inf_slot=None):
    n, k = X.shape
    Xn = torch.empty_like(X)
    w = _empty(k)
    _lib.call("bamg_test_weights", A.ref(), _p(X), n, k, -1 if inf_slot is None else int(inf_slot),
              _p(Xn), _p(w))
    return Xn, w


def fit_rows(adj, coarse_rank, X, w, caliber, radius, tol, constrain, nonneg, ridge=None):
    """Returns (cnt, col, val, (pinv_branch_fits, deferred_to_warp_path))."""
    n, k = X.shape
    cnt = _empty(n, I32)
    col = _empty(n * caliber, I32)
    val = _empty(n * caliber, F64)
    status = (C.c_int64 * 2)()
    _lib.call("bamg_fit_rows", adj.ref(), _p(coarse_rank), _p(X), _p(w), n, k, int(caliber),
              int(radius), float(tol), int(bool(constrain)), int(bool(nonneg)),
              -1.0 if ridge is None else float(ridge), _p(cnt), _p(col), _p(val), status)
    return cnt, col, val, (int(status[0]), int(status[1]))


def fit_rows_csr(adj, coarse_rank, X, w, caliber, radius, tol, constrain, nonneg, ncols, ridge=None):
    """fit_rows + rows_to_csr with one host read: (DeviceCSR, (pinv_branch_fits, deferred))."""
    n, k = X.shape
    cnt = _empty(n, I32)
    col = _empty(n * caliber, I32)
    val = _empty(n * caliber, F64)
    rp = _empty(n + 1, I32)
    status = (C.c_int64 * 2)()
    nnz = C.c_int64(0)
    _lib.call("bamg_fit_rows_csr", adj.ref(), _p(coarse_rank), _p(X), _p(w), n, k, int(caliber),
              int(radius), float(tol), int(bool(constrain)), int(bool(nonneg)),
              -1.0 if ridge is None else float(ridge), _p(cnt), _p(col), _p(val), _p(rp), status,
              C.byref(nnz))
    ci = _empty(max(nnz.value, 1), I32)
    va = _empty(max(nnz.value, 1), F64)
    _lib.call("bamg_rows_fill", _p(cnt), _p(col), _p(val), n, int(caliber), _p(rp), _p(ci), _p(va))
    return DeviceCSR(rp, ci[: nnz.value], va[: nnz.value], (n, ncols)), (int(status[0]), int(status[1]))


def fit_set_row_range(lo=None, hi=None):
    """Restrict the following LS fits to the fine points in rows [lo, hi) (None: every row)."""
    _lib.call("bamg_fit_set_row_range", -1 if lo is None else int(lo), -1 if hi is None else int(hi))


def fit_rows_csr_many(fits, raw=False):
    """Independent fits [dict(adj, coarse_rank, X, w, caliber, radius, tol,
    constrain, nonneg, ncols[, ridge])] (at most 4) with ONE host read for all
    of them: [(DeviceCSR, (pinv_branch_fits, deferred)), ...].  raw=True returns the
    fixed-stride rows [(cnt, col, val, caliber, ncols), ...] instead (the multi-GPU setup
    all-gathers them by rows before the CSR assembly)."""
    if not 1 <= len(fits) <= 4:
        raise ValueError("1..4 fits per batch")
    bufs = []
    for slot, f in enumerate(fits):
        X = f["X"]
        n, k = X.shape
        cal = int(f["caliber"])
        cnt = _empty(n, I32)
        col = _empty(n * cal, I32)
        val = _empty(n * cal, F64)
        rp = _empty(n + 1, I32)
        ridge = f.get("ridge")
        _lib.call("bamg_fit_rows_csr_slot", f["adj"].ref(), _p(f["coarse_rank"]), _p(X), _p(f["w"]), n, k, cal,
                  int(f["radius"]), float(f["tol"]), int(bool(f["constrain"])), int(bool(f["nonneg"])),
                  -1.0 if ridge is None else float(ridge), _p(cnt), _p(col), _p(val), _p(rp), slot)
        bufs.append((n, cal, cnt, col, val, rp, int(f["ncols"])))
    slots = (C.c_int32 * len(fits))(*range(len(fits)))
    status = (C.c_int64 * (2 * len(fits)))()
    nnz = (C.c_int64 * len(fits))()
    _lib.call("bamg_fit_rows_wait", len(fits), slots, status, nnz)
    if raw:
        return [(cnt, col, val, cal, ncols) for (n, cal, cnt, col, val, rp, ncols) in bufs]
    out = []
    for i, (n, cal, cnt, col, val, rp, ncols) in enumerate(bufs):
        m = int(nnz[i])
        ci = _empty(max(m, 1), I32)
        va = _empty(max(m, 1), F64)
        _lib.call("bamg_rows_fill", _p(cnt), _p(col), _p(val), n, cal, _p(rp), _p(ci), _p(va))
        out.append((DeviceCSR(rp, ci[:m], va[:m], (n, ncols)), (int(status[2 * i]), int(status[2 * i + 1]))))
    return out


def rows_to_csr(cnt, col, val, n, stride, ncols) -> DeviceCSR:
    rp = _empty(n + 1, I32)
    nnz = C.c_int64(0)
    _lib.call("bamg_rows_count", _p(cnt), _p(val), n, int(stride), _p(rp), C.byref(nnz))
    ci = _empty(max(nnz.value, 1), I32)
    va = _empty(max(nnz.value, 1), F64)
    _lib.call("bamg_rows_fill", _p(cnt), _p(col), _p(val), n, int(stride), _p(rp), _p(ci), _p(va))
    return DeviceCSR(rp, ci[: nnz.value], va[: nnz.value], (n, ncols))


# ----------------------------------------------------------------- coarsen
def axis_ranks(coord):
    n = coord.numel()
    rank = _empty(n, I32)
    nv = C.c_int64(0)
    _lib.call("bamg_axis_ranks", _p(coord), n, _p(rank), C.byref(nv))
    return rank, nv.value


def rerank(parent_rank, coarse_idx, nvalues_parent, exact=False):
    """Dense ranks of the coarse points' values.  The distinct-value count is
    only ever a buffer bound for the next rerank, so by default it is not read
    back (the parent's count bounds it; no host synchronisation)."""
    nc = coarse_idx.numel()
    out = _empty(nc, I32)
    nv = C.c_int64(0)
    _lib.call("bamg_rerank", _p(parent_rank), _p(coarse_idx), nc, int(nvalues_parent), _p(out),
              C.byref(nv) if exact else None)
    return out, (nv.value if exact else int(nvalues_parent))


def even_mask(ranks):
    n = ranks[0].numel()
    arr = (C.c_void_p * len(ranks))(*[r.data_ptr() for r in ranks])
    mask = _empty(n, U8)
    _lib.call("bamg_even_mask", arr, len(ranks), n, _p(mask))
    return mask


def split_from_mask(mask):
    n = mask.numel()
    coarse = _empty(n, I32)
    fine = _empty(n, I32)
    crank = _empty(n, I32)
    nc = C.c_int64(0)
    _lib.call("bamg_split_from_mask", _p(mask), n, _p(coarse), _p(fine), _p(crank), C.byref(nc))
    return coarse[: nc.value], fine[: n - nc.value], crank, nc.value


def cr_pass(A, adj, d, cmask, normals, n_fine, sweeps, omega, threshold, coarse_empty):
    ncand = C.c_int64(0)
    ncoarse = C.c_int64(0)
    _lib.call("bamg_cr_pass", A.ref(), adj.ref(), _p(d), _p(cmask), _p(normals), int(n_fine),
              int(sweeps), float(omega), float(threshold), int(bool(coarse_empty)), C.byref(ncand),
              C.byref(ncoarse))
    return ncand.value, ncoarse.value


# ------------------------------------------------------------------- dense
def csr_to_dense(A: DeviceCSR, transpose=False):
    """Column-major dense copy (torch tensor viewed as [cols][rows])."""
    n, m = A.shape
    D = _empty((m, n) if not transpose else (n, m))
    _lib.call("bamg_csr_to_dense", A.ref(), _p(D), n if not transpose else m, int(bool(transpose)))
    return D


def dense_pinv(Dcm, n, rank_tol=1e-12):
    Z = _empty((n, n))
    _lib.call("bamg_dense_pinv", _p(Dcm), n, float(rank_tol), _p(Z))
    return Z  # row-major pseudo-inverse


# ------------------------------------------------------ FOV diagnostics
def fov_points(Dcm, n, n_angles, tol=0.0):
    """Supporting points (re, im interleaved) of the angle sweep; Dcm column-major."""
    pts = _empty(2 * n_angles)
    it = C.c_int(0)
    _lib.call("bamg_fov_points", _p(Dcm), int(n), int(n_angles), float(tol), _p(pts), C.byref(it))
    return pts, it.value


def eigvals(Dcm, n):
    """(wr, wi) of a dense column-major matrix (unsorted)."""
    wr, wi = _empty(n), _empty(n)
    if _lib.call("bamg_eigvals", _p(Dcm), int(n), _p(wr), _p(wi)) == 2:
        raise np.linalg.LinAlgError("Eigenvalues did not converge")
    return wr, wi


def range_basis(Dcm, n, rank_tol):
    """(basis n x r, projected r x r) of a dense column-major matrix, as
    row-major torch views of the column-major results."""
    B = _empty(n * n)
    P = _empty(n * n)
    r = C.c_int(0)
    _lib.call("bamg_range_basis", _p(Dcm), int(n), float(rank_tol), _p(B), _p(P), C.byref(r))
    r = r.value
    return B[: n * r].view(r, n).T, P[: r * r].view(r, r).T


class CoarseLU:
    """The coarsest level's bordered LU kept on device by the implicit large
    path (bamg_coarse_lu): the V-cycle's coarsest solve goes through it."""

    def __init__(self, handle, n):
        self.handle = handle
        self.n = n
        self.shape = (n, n)

    def apply(self, b):
        x = _empty(self.n)
        bv = to_device_vec(b)
        _lib.call("bamg_coarse_lu_apply", self.handle, _p(bv), _p(x))
        return x

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().bamg_coarse_lu_destroy(_lib.ctx(), self.handle)
                self.handle = None
        except Exception:
            pass


def coarsest_triplets(Bd, Md, Nd, n, r, with_pinv=False):
    """(U, V, sigma, Z): with `with_pinv`, Z is B's row-major pseudo-inverse
    derived from the triplet solve's factors; None when not requested, when
    that path did not run or was not certified (the caller then builds it
    with dense_pinv)."""
    take = min(r, n)
    U = _empty((n, take))
    V = _empty((n, take))
    s = _empty(take)
    ok = C.c_int(0)
    lu = C.c_void_p()
    Z = _empty((n, n)) if with_pinv else None
    rc = _lib.call("bamg_coarsest_triplets_ex", _p(Bd), _p(Md), _p(Nd), n, take, _p(U), _p(V), _p(s),
                   _p(Z) if Z is not None else None, C.byref(ok), C.byref(lu))
    if rc == 2:
        raise ValueError("matrix is not positive definite (coarsest mass matrix)")
    if lu.value:
        return U, V, s, CoarseLU(lu, n)  # implicit large path: the kept LU serves the V-cycle
    return U, V, s, (Z if (Z is not None and ok.value) else None)


def coarsest_triplets_band(B: DeviceCSR, Bt: DeviceCSR, M: DeviceCSR, N: DeviceCSR, r, warm_right=None):
    """(U, V, sigma, CoarseLU) from the block-tridiagonal factorisations of the
    CSR operators (bamg_coarsest_band), or None when the level is not banded
    enough or the factorisation was not certified (dense path then)."""
    n = B.shape[0]
    take = min(r, n)
    U = _empty((n, take))
    V = _empty((n, take))
    s = _empty(take)
    lu = C.c_void_p()
    warm = None
    if warm_right is not None and tuple(warm_right.shape) == (n, take):
        warm = warm_right.contiguous()
    rc = _lib.call("bamg_coarsest_band", B.ref(), Bt.ref(), M.ref(), N.ref(), take, _p(warm), _p(U), _p(V), _p(s),
                   C.byref(lu))
    if rc != 0 or not lu.value:
        return None
    return U, V, s, CoarseLU(lu, n)


def uniform_draws(seed: int, k: int, n: int):
    """numpy default_rng(seed).random((k, n)) twice (right, then left) generated on
    the device (PCG64 jump-ahead, bit-identical), as n x k interleaved blocks."""
    import numpy as np
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    right = _empty((n, k))
    left = _empty((n, k))
    _lib.call("bamg_uniform_draws", s >> 64, s & m64, inc >> 64, inc & m64, int(k), int(n), _p(right), _p(left))
    return right, left


def sign_fix_l1(x, stride=1, uniform_fallback=False):
    n = x.shape[0]
    out = _empty(n)
    _lib.call("bamg_sign_fix_l1", _p(x), n, int(stride), _p(out), int(bool(uniform_fallback)))
    return out
