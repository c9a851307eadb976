"""Host-side geometry of the FOV diagnostics (fov.py: hull, origin distance,
point-in-polygon, bounds, CSV) against the reference's outputs in
tests/golden/fov.npz -- no GPU needed."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_1402_4005_b200.fov import (FovResult, _convex_hull, _origin_distance, elman_bound, fov_to_csv,
                                      nu_sidecar, point_in_fov, theorem2_bound)

GOLD = Path(__file__).resolve().parent / "golden" / "fov.npz"


@pytest.fixture(scope="module")
def g():
    with np.load(GOLD, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def test_hull_of_reference_hull_is_itself(g):
    """The reference's hull vertices are in convex position, counterclockwise
    from the lowest-x point: re-hulling them reproduces them exactly."""
    for name in g["names"]:
        b = g[f"{name}_boundary"]
        assert np.array_equal(_convex_hull(b), b), name


def test_hull_drops_interior_points(g):
    b = g["tandem7_boundary"]
    rng = np.random.default_rng(3)
    w = rng.random((40, b.size))  # strictly interior: convex combinations of the vertices
    w /= w.sum(axis=1, keepdims=True)
    pts = np.concatenate([b, w @ b])
    rng.shuffle(pts)
    h = _convex_hull(pts)
    assert h.size == b.size
    assert np.abs(h - b).max() <= 1e-14


def test_origin_distance_matches_reference(g):
    for name in g["names"]:
        nu, inside = _origin_distance(g[f"{name}_boundary"])
        assert nu == float(g[f"{name}_nu"]) and inside == bool(g[f"{name}_inside"]), name


def test_degenerate_hulls():
    assert _convex_hull(np.array([1 + 1j, 1 + 1j])).tolist() == [1 + 1j]
    assert _origin_distance(np.array([], dtype=complex)) == (np.inf, False)
    assert _origin_distance(np.array([3 + 4j])) == (5.0, False)
    seg = _convex_hull(np.array([-1.0 + 0j, 0.5 + 0j, 2.0 + 0j]))
    assert seg.tolist() == [-1 + 0j, 2 + 0j]
    assert _origin_distance(seg) == (0.0, False)


def test_point_in_fov_and_bounds(g):
    f = FovResult(boundary=g["diag30_boundary"], eigenvalues=g["diag30_eigenvalues"],
                  nu=float(g["diag30_nu"]), contains_origin=False)
    for lam in f.eigenvalues:
        assert point_in_fov(f, complex(lam), slack=1e-6)
    assert not point_in_fov(f, 0j)
    point = FovResult(boundary=np.array([1.0 + 0j]), eigenvalues=np.array([1.0 + 0j]), nu=1.0,
                      contains_origin=False)
    zero = FovResult(boundary=np.array([0.0 + 0j]), eigenvalues=np.array([0j]), nu=0.0, contains_origin=False)
    assert theorem2_bound(zero, point, 10) == 1.0
    assert theorem2_bound(point, point, 2) == 0.0
    assert elman_bound(point, 0.0, 3) == 1.0
    vals = [theorem2_bound(f, f, k) for k in (1, 2, 4, 8)]
    assert all(b <= a + 1e-15 for a, b in zip(vals, vals[1:]))


def test_csv_and_sidecar_format(g):
    import json
    f = FovResult(boundary=g["uniform8_boundary"], eigenvalues=g["uniform8_eigenvalues"],
                  nu=float(g["uniform8_nu"]), contains_origin=True)
    bcsv, ecsv = fov_to_csv(f)
    assert bcsv.splitlines()[0] == "re,im" and len(bcsv.splitlines()) == f.boundary.size + 1
    assert len(ecsv.splitlines()) == f.eigenvalues.size + 1
    assert json.loads(nu_sidecar({"nu": f.nu}))["nu"] == f.nu
