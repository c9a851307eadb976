"""Least-squares interpolation and restriction (mirrors markovmg/interp.py).

The per-fine-point greedy ridge least squares runs one THREAD per point in
csrc/interp.cu (compile-time trial sizes, points bucketed by candidate count);
points outside that path go to the warp-per-point Householder-QR kernel.  This
module keeps the reference's configuration objects and entry points and
assembles the fixed-stride row output into canonical CSR on device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from .coarsen import CfSplitting
from .device import DeviceCSR

WEIGHT_CAP = 1e16      # interp.py:23
WEIGHT_SPREAD = 1e4    # interp.py:27
RIDGE_KAPPA = 0.1      # interp.py:30
COEF_CAP = 10.0        # interp.py:33

#: levels below this many rows are fitted replicated on every rank (multi-GPU setup)
ROW_PARTITION_MIN_ROWS = 1 << 14
#: how many fits / sparse products of this process ran row-partitioned (tests, diagnostics)
PARTITION_STATS = {"fits": 0, "products": 0}


@dataclass(frozen=True)
class InterpConfig:
    """interp.py:36-58."""

    caliber: int = 2
    search_radius: int = 1
    constrain_constant_in_q: bool = True
    improvement_tol: float = 1e-3
    nonnegative: bool = True

    def __post_init__(self):
        if self.caliber < 1:
            raise ValueError("caliber must be at least 1")
        if self.search_radius not in (1, 2):
            raise ValueError("search_radius must be 1 or 2")


class WeightedTestSet:
    """Unit-norm test vectors (device, n x k interleaved) and weights (interp.py:61-79)."""

    def __init__(self, vectors, weights):
        self.dvectors = vectors     # n x k device
        self.dweights = weights     # k device (inf marks a constraint)

    @property
    def r(self) -> int:
        return int(self.dvectors.shape[1])

    @property
    def vectors(self) -> np.ndarray:
        """(k, n) host copy, the reference's layout."""
        return self.dvectors.cpu().numpy().T.copy()

    @property
    def weights(self) -> np.ndarray:
        return self.dweights.cpu().numpy()


def singular_test_weights(B, vectors, transpose_side: bool = False, infinite_slot=None,
                          Bt: DeviceCSR | None = None) -> WeightedTestSet:
    """Weights 1/||Bv||^2 (or 1/||B^T v||^2), capped (interp.py:82-102).

    `vectors` is an n x k device block (or the reference's (k, n) host array).
    """
    from .sparse import as_device
    A = as_device(B)
    if transpose_side:
        A = Bt if Bt is not None else engine.transpose(A)
    X = vectors
    if not isinstance(X, torch.Tensor):
        X = engine.to_device_vec(np.atleast_2d(np.asarray(vectors, dtype=np.float64)).T.copy())
    Xn, w = engine.test_weights(A, X.contiguous(), infinite_slot)
    return WeightedTestSet(Xn, w)


def _build_rows(adj: DeviceCSR, split: CfSplitting, tests: WeightedTestSet, cfg: InterpConfig,
                constrain: bool) -> DeviceCSR:
    """(n, n_c) operator: identity on C points, greedy LS rows on F points (interp.py:252-289)."""
    R, fallbacks = engine.fit_rows_csr(adj, split.dcrank, tests.dvectors, tests.dweights,
                                       cfg.caliber, cfg.search_radius, cfg.improvement_tol,
                                       constrain, cfg.nonnegative, split.n_coarse)
    return R


def build_interpolation(B, split: CfSplitting, tests: WeightedTestSet, cfg: InterpConfig,
                        adj: DeviceCSR | None = None) -> DeviceCSR:
    """P (interp.py:292-300)."""
    from .sparse import adjacency_structure
    S = adj if adj is not None else adjacency_structure(B)
    return _build_rows(S, split, tests, cfg, constrain=False)


def build_restriction_rows(B, split: CfSplitting, tests: WeightedTestSet, cfg: InterpConfig,
                           adj: DeviceCSR | None = None) -> DeviceCSR:
    """W = Q^T: rows fitted on B^T under the sum-to-one constraint (interp.py:312-313).

    pattern(B^T + B) == pattern(B + B^T), so the adjacency of B serves both.
    """
    from .sparse import adjacency_structure
    S = adj if adj is not None else adjacency_structure(B)
    return _build_rows(S, split, tests, cfg, constrain=cfg.constrain_constant_in_q)


def build_transfer_pair(B, split: CfSplitting, v_tests: WeightedTestSet, u_tests: WeightedTestSet,
                        cfg: InterpConfig, adj: DeviceCSR | None = None, comm=None):
    """(P, W): build_interpolation and build_restriction_rows of one level
    with one host synchronisation for both fits (they are independent).

    `comm` with more than one rank (multi-GPU setup): the per-point loop of _build_rows
    (interp.py:258-289) is independent per point, so every rank fits the fine points of its
    own contiguous row block (against the replicated test vectors and adjacency) and the
    fixed-stride rows are all-gathered before the CSR assembly: the same rows, bit for bit,
    as the single-GPU fit."""
    from .sparse import adjacency_structure
    S = adj if adj is not None else adjacency_structure(B)
    common = dict(adj=S, coarse_rank=split.dcrank, caliber=cfg.caliber, radius=cfg.search_radius,
                  tol=cfg.improvement_tol, nonneg=cfg.nonnegative, ncols=split.n_coarse)
    fits = [dict(common, X=v_tests.dvectors, w=v_tests.dweights, constrain=False),
            dict(common, X=u_tests.dvectors, w=u_tests.dweights, constrain=cfg.constrain_constant_in_q)]
    n = int(v_tests.dvectors.shape[0])
    if comm is not None and comm.world > 1 and n >= ROW_PARTITION_MIN_ROWS:
        from .distributed import RowPartition
        part = RowPartition(n, comm.world)
        r0, r1 = part.range(comm.rank)
        engine.fit_set_row_range(r0, r1)
        try:
            raw = engine.fit_rows_csr_many(fits, raw=True)
        finally:
            engine.fit_set_row_range(None)
        rows = [int(part.offsets[r + 1] - part.offsets[r]) for r in range(comm.world)]
        out = []
        for cnt, col, val, cal, ncols in raw:
            cnt_f = comm.all_gather_flat(cnt[r0:r1].contiguous(), rows)
            wide = [m * cal for m in rows]
            col_f = comm.all_gather_flat(col[r0 * cal:r1 * cal].contiguous(), wide)
            val_f = comm.all_gather_flat(val[r0 * cal:r1 * cal].contiguous(), wide)
            out.append(engine.rows_to_csr(cnt_f, col_f, val_f, n, cal, ncols))
            PARTITION_STATS["fits"] += 1
        return out[0], out[1]
    (P, _), (W, _) = engine.fit_rows_csr_many(fits)
    return P, W


def build_restriction(B, split: CfSplitting, tests: WeightedTestSet, cfg: InterpConfig,
                      adj: DeviceCSR | None = None) -> DeviceCSR:
    """Q = W^T (interp.py:303-314)."""
    return engine.transpose(build_restriction_rows(B, split, tests, cfg, adj))
