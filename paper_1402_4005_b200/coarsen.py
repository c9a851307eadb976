"""Coarse/fine splittings on device (mirrors markovmg/coarsen.py).

`CfSplitting` keeps the coarse list, fine list and coarse-rank map in HBM;
`.coarse` / `.fine` / `.coarse_rank` materialise host numpy copies on access.
Geometry is carried as per-axis ranks among distinct coordinate values
(`AxisRanks`), computed once on the finest level by the device radix sort
and re-ranked exactly on every coarse level (csrc/coarsen.cu).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from .device import DeviceCSR, device

MODES = ("geometric1d", "geometric2d", "cr")


class CfSplitting:
    """Disjoint coarse/fine index sets covering 0..n-1 (coarsen.py:23-52)."""

    def __init__(self, dcoarse, dfine, dcrank, n):
        self.dcoarse = dcoarse      # int32 device, ascending
        self.dfine = dfine          # int32 device, ascending
        self.dcrank = dcrank        # int32 device, -1 on F points
        self.n = int(n)
        self._host = {}
        if self.n_coarse == 0:
            raise ValueError("coarse set may not be empty")

    @classmethod
    def from_mask(cls, mask):
        """splitting_from_mask (coarsen.py:55-59); mask is a device uint8/bool tensor."""
        m = mask.to(torch.uint8) if mask.dtype != torch.uint8 else mask
        coarse, fine, crank, nc = engine.split_from_mask(m)
        return cls(coarse, fine, crank, m.numel())

    @property
    def n_coarse(self) -> int:
        return int(self.dcoarse.numel())

    def _h(self, key, t):
        if key not in self._host:
            self._host[key] = t.cpu().numpy().astype(np.int64)
        return self._host[key]

    @property
    def coarse(self) -> np.ndarray:
        return self._h("coarse", self.dcoarse)

    @property
    def fine(self) -> np.ndarray:
        return self._h("fine", self.dfine)

    @property
    def coarse_rank(self) -> np.ndarray:
        return self._h("crank", self.dcrank)

    def to_json(self) -> str:
        return json.dumps({"n": int(self.n), "coarse": self.coarse.tolist(),
                           "fine": self.fine.tolist()}, sort_keys=True)


def splitting_from_mask(coarse_mask) -> CfSplitting:
    if not isinstance(coarse_mask, torch.Tensor):
        coarse_mask = torch.from_numpy(np.asarray(coarse_mask, dtype=np.uint8)).to(device())
    return CfSplitting.from_mask(coarse_mask)


@dataclass(frozen=True)
class CoarseningConfig:
    """coarsen.py:62-81."""

    mode: str = "cr"
    stop_size: int = 500
    cr_sweeps: int = 5
    cr_threshold: float = 0.7
    max_levels: int = 20
    cr_omega: float = 0.7

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.stop_size < 2:
            raise ValueError("stop_size must be at least 2")
        if not 0.0 < self.cr_threshold < 1.0:
            raise ValueError("cr_threshold must lie in (0, 1)")
        if self.max_levels < 1:
            raise ValueError("max_levels must be positive")


class AxisRanks:
    """Per-axis ranks of the level's points among the distinct coordinate values.

    Level 0 ranks come from the host geometry (np.unique inverse, computed on
    device); coarse levels from `restrict(split)`.  `host` keeps the level's
    coordinates for lazy `Level.geometry` access.
    """

    def __init__(self, ranks, nvalues, host_coords=None):
        self.ranks = ranks          # list of int32 device tensors
        self.nvalues = nvalues      # list of distinct-value counts
        self.host_coords = host_coords

    @classmethod
    def from_geometry(cls, geometry):
        """`geometry`: host (n, d) array, or device per-axis coordinate columns
        (a d x n tensor) already resident in HBM."""
        if isinstance(geometry, torch.Tensor):
            cols = [geometry[a].contiguous() for a in range(geometry.shape[0])]
            host = None
        else:
            g = np.asarray(geometry, dtype=np.float64)
            if g.ndim != 2:
                raise ValueError("geometry must be an (n, d) array")
            cols = [torch.from_numpy(np.ascontiguousarray(g[:, a])).to(device()) for a in range(g.shape[1])]
            host = g
        ranks, nvals = [], []
        for col in cols:
            r, nv = engine.axis_ranks(col)
            ranks.append(r)
            nvals.append(nv)
        return cls(ranks, nvals, host)

    @property
    def ndim(self):
        return len(self.ranks)

    def restrict(self, split: CfSplitting) -> "AxisRanks":
        ranks, nvals = [], []
        for r, nv in zip(self.ranks, self.nvalues):
            rr, nn = engine.rerank(r, split.dcoarse, nv)
            ranks.append(rr)
            nvals.append(nn)
        host = None
        if self.host_coords is not None:
            host = _LazyRows(self.host_coords, split)
        return AxisRanks(ranks, nvals, host)


class _LazyRows:
    """geometry[split.coarse] materialised on first use."""

    def __init__(self, parent, split):
        self.parent, self.split = parent, split
        self._v = None

    def value(self):
        if self._v is None:
            base = self.parent.value() if isinstance(self.parent, _LazyRows) else self.parent
            self._v = base[self.split.coarse]
        return self._v


def geometric_coarsen(geometry, mode: str) -> CfSplitting:
    """Every other grid position per axis (coarsen.py:90-109)."""
    if geometry is None:
        raise ValueError("geometric coarsening needs coordinates")
    ranks = geometry if isinstance(geometry, AxisRanks) else AxisRanks.from_geometry(geometry)
    if mode == "geometric1d":
        use = ranks.ranks[:1]
    elif mode == "geometric2d":
        if ranks.ndim < 2:
            raise ValueError("2-D coarsening needs two coordinate columns")
        use = ranks.ranks[:2]
    else:
        raise ValueError(f"not a geometric mode: {mode!r}")
    mask = engine.even_mask(use)
    coarse, fine, crank, nc = engine.split_from_mask(mask)
    if nc == 0:
        raise ValueError("geometric coarsening produced an empty coarse set")
    return CfSplitting(coarse, fine, crank, mask.numel())


def cr_coarsen(B, cfg: CoarseningConfig, seed, adj: DeviceCSR | None = None,
               diag=None) -> CfSplitting:
    """Compatible-relaxation coarsening (coarsen.py:112-169).

    The seeded standard-normal draw per pass is made on the host from the
    same numpy generator as the reference (it defines the input); everything
    else -- F-relaxation, mu, candidates and the greedy MIS -- runs on device.
    """
    from .sparse import adjacency_structure, as_device
    A = as_device(B)
    n = A.shape[0]
    if engine.count_empty_rows(A):
        raise ValueError("matrix has an empty row")
    rng = np.random.default_rng(seed)
    S = adj if adj is not None else adjacency_structure(A)
    d = engine.diag(A) if diag is None else diag
    cmask = torch.zeros(n, dtype=torch.uint8, device=device())
    n_coarse = 0
    sweeps = max(cfg.cr_sweeps, 1)
    for _ in range(100):
        n_fine = n - n_coarse
        if n_fine == 0:
            break
        draw = torch.from_numpy(rng.standard_normal(n_fine)).to(device())
        ncand, n_coarse_new = engine.cr_pass(A, S, d, cmask, draw, n_fine, sweeps, cfg.cr_omega,
                                             cfg.cr_threshold, coarse_empty=(n_coarse == 0))
        if ncand == 0:
            if n_coarse == 0:
                n_coarse = n_coarse_new  # fallback point promoted on device
                continue
            break
        n_coarse = n_coarse_new
    if n_coarse == 0:
        cmask[0] = 1
    return CfSplitting.from_mask(cmask)


def make_splitting(B, geometry, cfg: CoarseningConfig, seed=None, adj=None, diag=None) -> CfSplitting:
    """coarsen.py:172-176."""
    if cfg.mode in ("geometric1d", "geometric2d"):
        return geometric_coarsen(geometry, cfg.mode)
    return cr_coarsen(B, cfg, seed, adj=adj, diag=diag)
