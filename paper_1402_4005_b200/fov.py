"""Field-of-values boundaries, range projections and GMRES residual bounds
(mirrors markovmg/fov.py).

The dense work runs on device (csrc/fov.cu through the C ABI):

* the angle sweep of `fov_boundary` -- every angle's top eigenvector of the
  Hermitian part of e^{i theta} M, all angles in one batched Lanczos whose
  operator applications are one DMMA GEMM per step (fov.py:85-115);
* `eigenvalue_dots` -- balancing, Householder Hessenberg reduction and the
  Francis double-shift QR iteration (fov.py:60-67, LAPACK dgeev there);
* the SVD range basis and the projected operator of `project_range` /
  `projected_preconditioned` -- one-sided Jacobi SVD and two GEMMs
  (fov.py:194-223); the preconditioned columns C B e_j are V-cycle applies on
  device when `precond` is this package's VCycleOperator.

What stays on the host is geometry on at most `n_angles` points (the convex
hull, the distance to the origin, point-in-polygon), the scalar bounds and the
CSV / JSON formatting -- the reference's own host logic, restated.

Inputs are real (every caller in the reference passes chain matrices or their
real projections); a matrix with a non-zero imaginary part is rejected with a
ValueError.  Same names, arguments, cap and error behaviour as the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from .device import DeviceCSR, device

DENSE_CAP = 1200


@dataclass
class FovResult:
    """Convex boundary polygon, eigenvalue dots, and the distance to the origin."""

    boundary: np.ndarray
    eigenvalues: np.ndarray
    nu: float
    contains_origin: bool


@dataclass
class ProjectedSystem:
    """Orthonormal range basis and the projected operator."""

    basis: np.ndarray
    projected: np.ndarray


def _check_cap(n: int, cap: int):
    if n > cap:
        raise ValueError(f"dense analysis is capped at n = {cap}; "
                         f"got {n} (use a smaller instance)")


def _host_real(A) -> np.ndarray:
    A = np.asarray(A)
    if np.iscomplexobj(A):
        if np.abs(A.imag).max(initial=0.0) != 0.0:
            raise ValueError("the device field-of-values path takes real matrices")
        A = A.real
    return np.asarray(A, dtype=np.float64)


def _columns_to_device(cols, n):
    """Stack n column vectors (host or device) into a column-major device block."""
    D = torch.empty((n, n), dtype=torch.float64, device=device())
    for j, c in enumerate(cols):
        if isinstance(c, torch.Tensor):
            D[j] = c.to(device=D.device, dtype=torch.float64)
        else:
            D[j] = torch.from_numpy(_host_real(c).reshape(-1))
    return D


def _dense_device(M, n: int | None = None, cap: int | None = None):
    """(column-major device matrix as a (cols, rows) tensor, n) of a dense
    array, scipy sparse matrix, DeviceCSR, device tensor or matrix-free
    callable (fov.py:41-50 `_as_dense`)."""
    if isinstance(M, DeviceCSR):
        if M.shape[0] != M.shape[1]:
            raise ValueError(f"expected a square matrix, got shape {M.shape}")
        if cap is not None:
            _check_cap(M.shape[0], cap)
        return engine.csr_to_dense(M), M.shape[0]
    if hasattr(M, "toarray"):
        M = M.toarray()
    if callable(M) and not isinstance(M, (np.ndarray, torch.Tensor)):
        if n is None:
            raise ValueError("matrix-free operators need an explicit dimension")
        if cap is not None:
            _check_cap(n, cap)
        return _columns_to_device((M(col) for col in np.eye(n)), n), n
    if isinstance(M, torch.Tensor):
        if M.dim() != 2 or M.shape[0] != M.shape[1]:
            raise ValueError(f"expected a square matrix, got shape {tuple(M.shape)}")
        if cap is not None:
            _check_cap(M.shape[0], cap)
        return M.to(device=device(), dtype=torch.float64).T.contiguous(), M.shape[0]
    A = _host_real(M)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {A.shape}")
    if cap is not None:
        _check_cap(A.shape[0], cap)
    return torch.from_numpy(np.ascontiguousarray(A.T)).to(device()), A.shape[0]


def _eigvals_device(D, n) -> np.ndarray:
    wr, wi = engine.eigvals(D, n)
    vals = wr.cpu().numpy() + 1j * wi.cpu().numpy()
    order = np.lexsort((vals.imag, vals.real))
    return vals[order]


def eigenvalue_dots(M) -> np.ndarray:
    """Full spectrum of a dense matrix, sorted by (real, imag) (fov.py:60-67)."""
    D, n = _dense_device(M, cap=DENSE_CAP)
    return _eigvals_device(D, n)


def fov_boundary(M, n_angles: int = 256, n: int | None = None,
                 dense_cap: int = DENSE_CAP) -> FovResult:
    """Trace the field-of-values boundary with an angle sweep (fov.py:85-115).

    Angle t contributes the supporting point <Mv, v> of the top eigenvector v
    of the Hermitian part of e^{i 2 pi t / n_angles} M; the boundary is the
    convex hull of the points and `nu` its distance to the origin (zero when
    the origin lies inside)."""
    if n_angles < 16:
        raise ValueError("need at least 16 angles")
    D, dim = _dense_device(M, n, cap=dense_cap)
    pts, _ = engine.fov_points(D, dim, n_angles)
    p = pts.cpu().numpy()
    points = p[0::2] + 1j * p[1::2]
    hull = _convex_hull(points)
    nu, inside = _origin_distance(hull)
    _check_cap(dim, DENSE_CAP)
    eigs = _eigvals_device(D, dim)
    return FovResult(boundary=hull, eigenvalues=eigs, nu=nu, contains_origin=inside)


def _cross(o, a, b) -> float:
    return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])


def _convex_hull(points: np.ndarray) -> np.ndarray:
    """Counterclockwise convex hull of complex points, Andrew's monotone chain
    on the points rounded to 15 decimals; collinear points are dropped
    (fov.py:118-141)."""
    uniq = np.unique(np.round(np.asarray(points, dtype=np.complex128), 15))
    xy = sorted(zip(uniq.real.tolist(), uniq.imag.tolist()))
    if len(xy) <= 2:
        return np.array([complex(a, b) for a, b in xy])

    def chain(seq):
        out = []
        for q in seq:
            while len(out) >= 2 and _cross(out[-2], out[-1], q) <= 0:
                out.pop()
            out.append(q)
        return out

    lower, upper = chain(xy), chain(xy[::-1])
    ring = lower[:-1] + upper[:-1]
    if not ring:
        ring = [xy[0], xy[-1]]
    return np.array([complex(a, b) for a, b in ring])


def _origin_distance(hull: np.ndarray) -> tuple[float, bool]:
    """Distance of the polygon to 0 and whether 0 is strictly inside (fov.py:144-167)."""
    if hull.size == 0:
        return np.inf, False
    if hull.size == 1:
        return float(abs(hull[0])), False
    P = np.column_stack([hull.real, hull.imag])
    m = len(P)
    edges = m if m >= 3 else 1
    best = np.inf
    inside = m >= 3
    for k in range(edges):
        a, b = P[k], P[(k + 1) % m]
        e = b - a
        ee = float(e @ e)
        t = 0.0 if ee == 0.0 else float(np.clip(-(a @ e) / ee, 0.0, 1.0))
        best = min(best, float(np.hypot(*(a + t * e))))
        if m >= 3 and e[0] * (-a[1]) - e[1] * (-a[0]) < 0.0:
            inside = False
    return (0.0, True) if inside else (best, False)


def point_in_fov(fov: FovResult, z: complex, slack: float = 1e-8) -> bool:
    """Whether z lies in the boundary polygon, allowing `slack` outside (fov.py:170-191)."""
    hull = fov.boundary
    if hull.size == 0:
        return False
    if hull.size <= 2:
        a = np.array([hull[0].real, hull[0].imag])
        b = np.array([hull[-1].real, hull[-1].imag])
        p = np.array([z.real, z.imag])
        e = b - a
        ee = float(e @ e)
        t = 0.0 if ee == 0.0 else float(np.clip(((p - a) @ e) / ee, 0.0, 1.0))
        return float(np.hypot(*(a + t * e - p))) <= slack
    P = np.column_stack([hull.real, hull.imag])
    m = len(P)
    scale = max(np.abs(P).max(), 1.0)
    for k in range(m):
        a, b = P[k], P[(k + 1) % m]
        e = b - a
        side = e[0] * (z.imag - a[1]) - e[1] * (z.real - a[0])
        if side < -slack * scale * max(np.hypot(*e), 1e-300):
            return False
    return True


def _project(D, n, rank_tol) -> ProjectedSystem:
    basis, projected = engine.range_basis(D, n, rank_tol)
    return ProjectedSystem(basis=basis.cpu().numpy(), projected=projected.cpu().numpy())


def project_range(B, rank_tol: float = 1e-12, dense_cap: int = DENSE_CAP) -> ProjectedSystem:
    """Project B onto an orthonormal basis of its range (fov.py:194-207): the
    left singular vectors with sigma > rank_tol sigma_max, descending."""
    D, n = _dense_device(B, cap=dense_cap)
    return _project(D, n, rank_tol)


def projected_preconditioned(B, precond, rank_tol: float = 1e-12,
                             dense_cap: int = DENSE_CAP) -> ProjectedSystem:
    """Materialize the preconditioned operator CB and project onto its range
    (fov.py:210-221).  With this package's VCycleOperator the columns C B e_j
    are V-cycle applies on device; any other callable gets host columns."""
    n = B.shape[0]
    _check_cap(n, dense_cap)
    D, _ = _dense_device(B)
    apply = precond.apply if hasattr(precond, "apply") else precond
    on_device = hasattr(precond, "handle")
    if on_device:
        cols = (apply(D[j].clone()) for j in range(n))
    else:
        Bh = D.T.cpu().numpy()
        cols = (np.asarray(apply(Bh[:, j])) for j in range(n))
    CB = _columns_to_device(cols, n)
    return _project(CB, n, rank_tol)


def theorem2_bound(fov_m: FovResult, fov_minv: FovResult, k: int) -> float:
    """Residual reduction factor (1 - nu(F(M)) nu(F(M^-1)))^(k/2), clamped to
    [0, 1] (fov.py:224-234)."""
    base = min(max(1.0 - fov_m.nu * fov_minv.nu, 0.0), 1.0)
    return float(base ** (k / 2.0))


def elman_bound(fov_m: FovResult, norm_m: float, k: int) -> float:
    """The classical variant (1 - (nu / ||M||)^2)^(k/2) (fov.py:237-243)."""
    if norm_m <= 0.0:
        return 1.0
    base = min(max(1.0 - (fov_m.nu / norm_m) ** 2, 0.0), 1.0)
    return float(base ** (k / 2.0))


def fov_to_csv(fov: FovResult) -> tuple[str, str]:
    """Plot-ready CSV bodies: boundary points and eigenvalue dots (fov.py:246-254)."""
    def body(zs):
        return "\n".join(["re,im"] + [f"{z.real!r},{z.imag!r}" for z in zs]) + "\n"
    return body(fov.boundary), body(fov.eigenvalues)


def nu_sidecar(values: dict) -> str:
    return json.dumps({k: float(v) for k, v in values.items()}, indent=2, sort_keys=True)
