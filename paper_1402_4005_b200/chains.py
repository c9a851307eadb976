"""Benchmark Markov chains as host inputs (the reference's chains.py is input
generation, out of the hot path; these generators produce the SAME canonical
CSR of B = I - A, bit for bit, vectorised so the 16.8M-state tandem chain
builds in seconds).

Tandem and uniform lattices are assembled directly in CSR form from their
stencils; the self-loop masses are accumulated in the reference's order
(chains.py:157-172) so every value matches.  Random planar chains triangulate
with scipy's Qhull Delaunay instead of the reference's O(n^2) Bowyer-Watson
(SURVEY.md section 8(d)); birth-death and Petri-net chains follow the
reference's constructions.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np
from scipy import sparse as sp

from .sparse import make_csr

FAMILIES = ("birth-death", "uniform2d", "tandem", "planar", "petri", "imported")


@dataclass(frozen=True)
class ChainProblem:
    """Column-stochastic A, B = I - A and metadata (chains.py:26-36)."""

    A: object
    B: object
    n: int
    family: str
    params: dict
    geometry: np.ndarray | None = None
    seed: int | None = None
    # optional torch.cuda.Event: a device `geometry` tensor still being copied in on another
    # stream is ready once it has fired (run_setup waits on it right before the first split,
    # so the upload overlaps the initial relaxation)
    geometry_ready: object = None
    # the same for a device operator B whose arrays are still in flight: run_setup draws the seeded
    # test vectors first and waits on this event before it first touches B
    B_ready: object = None


def _finish(A, family, params, geometry=None, seed=None, validate=True) -> ChainProblem:
    """Validate stochasticity / irreducibility and form B (chains.py:39-61)."""
    A = make_csr(A)
    n = A.shape[0]
    if validate:
        from scipy.sparse.csgraph import connected_components
        if A.shape[0] != A.shape[1]:
            raise ValueError("transition matrix must be square")
        if A.nnz and A.data.min() < 0.0:
            raise ValueError("transition matrix has negative entries")
        colsums = np.asarray(A.sum(axis=0)).ravel()
        worst = int(np.argmax(np.abs(colsums - 1.0)))
        if abs(colsums[worst] - 1.0) > 1e-12:
            raise ValueError(f"columns do not sum to one: worst column {worst} sums to {colsums[worst]:.16g}")
        ncomp, labels = connected_components(A, directed=True, connection="strong")
        if ncomp != 1:
            raise ValueError(f"chain is reducible: {ncomp} strongly connected components")
    B = make_csr(sp.eye_array(n, format="csr", dtype=np.float64) - A)
    return ChainProblem(A=A, B=B, n=n, family=family, params=dict(params), geometry=geometry, seed=seed)


def _csr_from_stencil(n, cols_list, vals_list):
    """Assemble a CSR whose row i holds (cols_list[t][i], vals_list[t][i]) for
    every stencil slot t with cols >= 0, slots already in ascending column order."""
    cols = np.stack(cols_list, axis=1)
    vals = np.stack(vals_list, axis=1)
    keep = cols >= 0
    counts = keep.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return sp.csr_array((vals[keep], cols[keep].astype(np.int32), indptr.astype(np.int32)), shape=(n, n))


def tandem_queue(side: int, lam: float = 11.0 / 31.0, mu1: float = 10.0 / 31.0,
                 mu2: float = 10.0 / 31.0, with_A: bool = True, validate: bool = True) -> ChainProblem:
    """Two queues in series on a side x side grid, node = q2*side + q1 (chains.py:134-179)."""
    if side < 2:
        raise ValueError("side must be at least 2")
    if abs(lam + mu1 + mu2 - 1.0) > 1e-12:
        raise ValueError("transition probabilities must sum to 1")
    n = side * side
    idx = np.arange(n, dtype=np.int64)
    q1 = idx % side
    q2 = idx // side
    # self-loop mass of source j, accumulated in the reference's order
    stay = np.zeros(n)
    stay = np.where(q1 + 1 > side - 1, stay + lam, stay)
    stay = np.where(~((q1 >= 1) & (q2 + 1 <= side - 1)), stay + mu1, stay)
    stay = np.where(q2 < 1, stay + mu2, stay)
    # row i of A collects sources j -> i: (q1+1, q2-1) via mu1 [col i-side+1],
    # (q1-1, q2) via lam [col i-1], self [col i], (q1, q2+1) via mu2 [col i+side]
    c_mu1 = np.where((q1 + 1 <= side - 1) & (q2 >= 1), idx - side + 1, -1)
    c_lam = np.where(q1 >= 1, idx - 1, -1)
    c_self = np.where(stay > 0.0, idx, -1)
    c_mu2 = np.where(q2 + 1 <= side - 1, idx + side, -1)
    ones = np.ones(n)
    A = _csr_from_stencil(n, [c_mu1, c_lam, c_self, c_mu2], [mu1 * ones, lam * ones, stay, mu2 * ones])
    # B = I - A in canonical form: 1 - a_ii on the diagonal (1.0 where no self loop)
    d = np.where(stay > 0.0, 1.0 - stay, 1.0)
    c_diag = np.where(d != 0.0, idx, -1)
    B = _csr_from_stencil(n, [c_mu1, c_lam, c_diag, c_mu2], [-mu1 * ones, -lam * ones, d, -mu2 * ones])
    geometry = np.column_stack([q1.astype(np.float64), q2.astype(np.float64)])
    params = {"side": side, "n": n, "lambda": lam, "mu1": mu1, "mu2": mu2}
    if validate:
        ref = _finish(A, "tandem", params, geometry=geometry)
        return ChainProblem(A=ref.A, B=B, n=n, family="tandem", params=params, geometry=geometry)
    return ChainProblem(A=A if with_A else None, B=B, n=n, family="tandem", params=params,
                        geometry=geometry)


def uniform_2d(side: int, validate: bool = True) -> ChainProblem:
    """Random walk on a side x side lattice, node = iy*side + ix (chains.py:95-131)."""
    if side < 2:
        raise ValueError("side must be at least 2")
    n = side * side
    idx = np.arange(n, dtype=np.int64)
    ix = idx % side
    iy = idx // side
    deg = (ix > 0).astype(np.int64) + (ix < side - 1) + (iy > 0) + (iy < side - 1)
    p = 1.0 / deg  # probability of leaving node j to each neighbour
    c_s = np.where(iy > 0, idx - side, -1)
    c_w = np.where(ix > 0, idx - 1, -1)
    c_e = np.where(ix < side - 1, idx + 1, -1)
    c_n = np.where(iy < side - 1, idx + side, -1)
    pick = lambda c: p[np.where(c >= 0, c, 0)]  # A_ij = p_j for neighbour j of i
    A = _csr_from_stencil(n, [c_s, c_w, c_e, c_n], [pick(c_s), pick(c_w), pick(c_e), pick(c_n)])
    c_d = idx
    B = _csr_from_stencil(n, [c_s, c_w, c_d, c_e, c_n],
                          [-pick(c_s), -pick(c_w), np.ones(n), -pick(c_e), -pick(c_n)])
    geometry = np.column_stack([ix.astype(np.float64), iy.astype(np.float64)])
    params = {"side": side, "n": n}
    if validate:
        ref = _finish(A, "uniform2d", params, geometry=geometry)
        return ChainProblem(A=ref.A, B=B, n=n, family="uniform2d", params=params, geometry=geometry)
    return ChainProblem(A=A, B=B, n=n, family="uniform2d", params=params, geometry=geometry)


def lattice_chain_device(family: str, side: int, lam: float = 11.0 / 31.0, mu1: float = 10.0 / 31.0,
                         mu2: float = 10.0 / 31.0) -> ChainProblem:
    """The tandem / uniform2d chain's B assembled directly in HBM
    (csrc/chains.cu): the same canonical CSR as tandem_queue / uniform_2d,
    bit for bit, without the host matrix or its upload.  A is not formed
    (`A=None`); geometry is the device (2, n) per-axis block the setup takes."""
    import ctypes as C

    import torch

    from . import _lib
    from .device import DeviceCSR, device
    if family not in ("tandem", "uniform2d"):
        raise ValueError("device assembly covers the tandem and uniform2d lattices")
    if side < 2:
        raise ValueError("side must be at least 2")
    if family == "tandem" and abs(lam + mu1 + mu2 - 1.0) > 1e-12:
        raise ValueError("transition probabilities must sum to 1")
    fid = 0 if family == "tandem" else 1
    n = side * side
    dev = device()
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    geo = torch.empty((2, n), dtype=torch.float64, device=dev)
    nnz = C.c_int64(0)
    _lib.call("bamg_chain_lattice_count", fid, side, float(lam), float(mu1), float(mu2), _lib.ptr(rp),
              _lib.ptr(geo), C.byref(nnz))
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
    _lib.call("bamg_chain_lattice_fill", fid, side, float(lam), float(mu1), float(mu2), _lib.ptr(rp),
              _lib.ptr(ci), _lib.ptr(va))
    B = DeviceCSR(rp, ci[: nnz.value], va[: nnz.value], (n, n))
    params = {"side": side, "n": n}
    if family == "tandem":
        params.update({"lambda": lam, "mu1": mu1, "mu2": mu2})
    return ChainProblem(A=None, B=B, n=n, family=family, params=params, geometry=geo)


def planar_chain_device(n: int, seed: int = 1) -> ChainProblem:
    """The random planar chain's B assembled in HBM from the Delaunay triangles
    (csrc/chains.cu): the same point draw as random_planar / the reference
    (chains.py:279-280), Qhull on the host, then degrees, de-duplicated
    neighbour lists and the canonical CSR of I - A on the device -- bit for bit
    random_planar's B without the host matrix or its upload.  A is not formed."""
    import ctypes as C

    import torch
    from scipy.spatial import Delaunay

    from . import _lib
    from .device import DeviceCSR, device
    if n < 4:
        raise ValueError("need at least four points")
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    pts = rng.random((n, 2))
    tri = np.ascontiguousarray(Delaunay(pts).simplices, dtype=np.int32)
    dev = device()
    dtri = torch.from_numpy(tri).to(dev)
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    nnz = C.c_int64(0)
    _lib.call("bamg_chain_planar_count", _lib.ptr(dtri), tri.shape[0], n, _lib.ptr(rp), C.byref(nnz))
    ci = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    va = torch.empty(nnz.value, dtype=torch.float64, device=dev)
    _lib.call("bamg_chain_planar_fill", _lib.ptr(dtri), tri.shape[0], n, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va))
    B = DeviceCSR(rp, ci, va, (n, n))
    geo = torch.from_numpy(np.ascontiguousarray(pts.T)).to(dev)
    return ChainProblem(A=None, B=B, n=n, family="planar", params={"n": n}, geometry=geo, seed=seed)


def birth_death(n: int, mu: float = 0.96) -> ChainProblem:
    """Biased walk on a path (chains.py:64-92)."""
    if n < 2:
        raise ValueError("need at least two states")
    if not 0.0 < mu < 1.0:
        raise ValueError("mu must lie strictly between 0 and 1")
    rows, cols, vals = [], [], []
    for j in range(n):
        if j == 0:
            rows += [1, 0]
            cols += [0, 0]
            vals += [mu, 1.0 - mu]
        elif j == n - 1:
            rows += [n - 2, n - 1]
            cols += [j, j]
            vals += [1.0 - mu, mu]
        else:
            rows += [j + 1, j - 1]
            cols += [j, j]
            vals += [mu, 1.0 - mu]
    A = make_csr(sp.coo_array((np.asarray(vals), (np.asarray(rows), np.asarray(cols))), shape=(n, n)))
    geometry = np.arange(n, dtype=np.float64).reshape(n, 1)
    return _finish(A, "birth-death", {"n": n, "mu": mu}, geometry=geometry)


def random_planar(n: int, seed: int = 1, validate: bool = True) -> ChainProblem:
    """Walk on the Delaunay triangulation of n uniform points (chains.py:270-302).

    Same point draw as the reference (default_rng(SeedSequence(seed)).random);
    the triangulation is scipy's Qhull (the reference's Bowyer-Watson is O(n^2)).
    """
    from scipy.spatial import Delaunay
    if n < 4:
        raise ValueError("need at least four points")
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    pts = rng.random((n, 2))
    tri = Delaunay(pts)
    s = tri.simplices
    e = np.concatenate([s[:, [0, 1]], s[:, [1, 2]], s[:, [0, 2]]])
    e = np.sort(e, axis=1)
    e = np.unique(e, axis=0)
    a, b = e[:, 0], e[:, 1]
    deg = np.bincount(a, minlength=n) + np.bincount(b, minlength=n)
    if deg.min() == 0:
        raise ValueError("triangulation left an isolated point")
    rows = np.concatenate([b, a])
    cols = np.concatenate([a, b])
    vals = np.concatenate([1.0 / deg[a], 1.0 / deg[b]])
    A = make_csr(sp.coo_array((vals, (rows, cols)), shape=(n, n)))
    return _finish(A, "planar", {"n": n}, geometry=pts, seed=seed, validate=validate)


def molloy_net(tokens: int):
    """Five-place fork/join net (chains.py:334-353) as (places, transitions, marking)."""
    if tokens < 1:
        raise ValueError("need at least one token")
    transitions = (({0: 1}, {1: 1, 2: 1}, 1.0), ({1: 1}, {3: 1}, 1.0), ({2: 1}, {4: 1}, 1.0),
                   ({3: 1}, {1: 1}, 1.0), ({3: 1, 4: 1}, {0: 1}, 1.0))
    return (5, transitions, (tokens, 0, 0, 0, 0))


def petri_reachability(spec, state_cap: int = 10 ** 6) -> ChainProblem:
    """Chain on the reachable markings, breadth-first order (chains.py:381-423)."""
    places, transitions, marking = spec
    initial = tuple(marking)
    index = {initial: 0}
    order = [initial]
    queue = deque([initial])
    rows, cols, vals = [], [], []
    while queue:
        m = queue.popleft()
        j = index[m]
        enabled = []
        for inp, out, w in transitions:
            if all(m[p] >= need for p, need in inp.items()):
                nxt = list(m)
                for p, need in inp.items():
                    nxt[p] -= need
                for p, add in out.items():
                    nxt[p] += add
                enabled.append((tuple(nxt), w))
        if not enabled:
            raise ValueError(f"deadlock: marking {m} enables no transition (chain not irreducible)")
        wsum = sum(w for _, w in enabled)
        for nxt, w in enabled:
            if nxt not in index:
                if len(index) >= state_cap:
                    raise ValueError(f"reachability set exceeds the state cap of {state_cap}")
                index[nxt] = len(order)
                order.append(nxt)
                queue.append(nxt)
            rows.append(index[nxt])
            cols.append(j)
            vals.append(w / wsum)
    n = len(order)
    A = make_csr(sp.coo_array((np.asarray(vals, dtype=np.float64), (np.asarray(rows), np.asarray(cols))),
                              shape=(n, n)))
    return _finish(A, "petri", {"places": places, "n_transitions": len(transitions),
                                "initial_marking": list(marking), "n": n})


def petri_spec_from_json(text: str):
    """Petri net from JSON {places, transitions: [{inputs, outputs, weight}], initial_marking}
    (chains.py:370-378), as the (places, transitions, marking) tuple petri_reachability takes."""
    import json
    doc = json.loads(text)
    transitions = tuple(({int(k): int(v) for k, v in t["inputs"].items()},
                         {int(k): int(v) for k, v in t["outputs"].items()},
                         float(t.get("weight", 1.0))) for t in doc["transitions"])
    return (int(doc["places"]), transitions, tuple(int(x) for x in doc["initial_marking"]))


def import_chain(path) -> ChainProblem:
    """Chain from a Matrix Market file holding A or B = I - A, told apart by the
    column sums (near one: stochastic A; near zero: B) (chains.py:426-447)."""
    from .sparse import load_matrix_market
    M = load_matrix_market(path)
    if M.shape[0] != M.shape[1]:
        raise ValueError("imported matrix must be square")
    colsums = np.asarray(M.sum(axis=0)).ravel()
    if np.abs(colsums - 1.0).max(initial=0.0) <= 1e-8:
        A = M
    elif np.abs(colsums).max(initial=0.0) <= 1e-8:
        A = make_csr(sp.eye_array(M.shape[0], format="csr", dtype=np.float64) - M)
    else:
        worst = int(np.argmax(np.minimum(np.abs(colsums - 1.0), np.abs(colsums))))
        raise ValueError(f"file is neither column-stochastic nor zero-column-sum: column {worst} "
                         f"sums to {colsums[worst]:.16g}")
    return _finish(A, "imported", {"path": str(path)})


def make_chain(family: str, **kw) -> ChainProblem:
    """chains.py:450-464."""
    if family == "birth-death":
        return birth_death(kw["n"], kw.get("mu", 0.96))
    if family == "uniform2d":
        return uniform_2d(kw["side"], validate=kw.get("validate", True))
    if family == "tandem":
        return tandem_queue(kw["side"], kw.get("lam", 11.0 / 31.0), kw.get("mu1", 10.0 / 31.0),
                            kw.get("mu2", 10.0 / 31.0), validate=kw.get("validate", True))
    if family == "planar":
        return random_planar(kw["n"], kw.get("seed", 1), validate=kw.get("validate", True))
    if family == "petri":
        return petri_reachability(kw.get("spec") or molloy_net(kw["tokens"]), kw.get("state_cap", 10 ** 6))
    raise ValueError(f"unknown family {family!r}")
