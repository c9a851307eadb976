"""Adaptive multilevel setup (mirrors markovmg/bootstrap.py, Algorithm 1).

The recursion, stop/stall/truncation rules and seed bookkeeping are host
control flow on scalars, exactly as in the reference; every array operation
is an engine launch on device-resident data:
  smoothing blocks (csrc/setup.cu), test weights and LS transfer rows
  (csrc/interp.cu), Galerkin products (csrc/spgemm.cu), C/F splits
  (csrc/coarsen.cu), coarsest triplets (csrc/dense.cu).
Test vectors are n x k interleaved device blocks; `TripletSet.left/right`
give the reference's (k, n) host layout on access.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, engine
from .coarsen import AxisRanks, CfSplitting, CoarseningConfig, make_splitting
from .device import DeviceCSR, device
from .interp import InterpConfig, build_transfer_pair, singular_test_weights
from .relax import SmootherConfig
from .sparse import adjacency_structure, as_device

#: bootstrap.py:329
SICK_DIAG_FRACTION = 0.02

_DEBUG = bool(os.environ.get("BAMG_DEBUG"))

#: optional phase profiler (bench.py --breakdown): name -> seconds.  Each
#: phase boundary synchronises the device, so it is off on the timed path.
PHASES: dict | None = None
#: optional sync-free phase recorder (tools/timeline.py): called with
#: (name, entering) at every phase boundary.
RECORDER = None


class _phase:
    def __init__(self, name, level=None):
        self.name = name
        self.level = level

    def __enter__(self):
        _lib.nvtx_push(f"bamg.setup.{self.name}" if self.level is None else f"bamg.setup.L{self.level}.{self.name}")
        if RECORDER is not None:
            RECORDER(self.name, True)
        if PHASES is not None:
            torch.cuda.synchronize()
            self.t = time.perf_counter()

    def __exit__(self, *exc):
        if RECORDER is not None:
            RECORDER(self.name, False)
        if PHASES is not None:
            torch.cuda.synchronize()
            PHASES[self.name] = PHASES.get(self.name, 0.0) + time.perf_counter() - self.t
        _lib.nvtx_pop()


class TripletSet:
    """Approximate singular triplets on device (bootstrap.py:35-59)."""

    def __init__(self, sigmas, left, right):
        self.dsigmas = sigmas   # k, device
        self.dleft = left       # n x k, device
        self.dright = right     # n x k, device
        if not (self.dsigmas.numel() == self.dleft.shape[1] == self.dright.shape[1]):
            raise ValueError("inconsistent triplet counts")

    @property
    def r(self) -> int:
        return int(self.dsigmas.numel())

    @property
    def n(self) -> int:
        return int(self.dright.shape[0])

    @property
    def sigmas(self) -> np.ndarray:
        return self.dsigmas.cpu().numpy()

    @property
    def left(self) -> np.ndarray:
        return self.dleft.cpu().numpy().T.copy()

    @property
    def right(self) -> np.ndarray:
        return self.dright.cpu().numpy().T.copy()

    def copy(self) -> "TripletSet":
        return TripletSet(self.dsigmas.clone(), self.dleft.clone(), self.dright.clone())


@dataclass(frozen=True)
class SetupConfig:
    """bootstrap.py:62-80."""

    n_tests: int = 8
    setup_cycles: int = 1
    inner_passes: int = 1
    smoother: SmootherConfig = field(default_factory=SmootherConfig)
    interp: InterpConfig = field(default_factory=InterpConfig)
    coarsening: CoarseningConfig = field(default_factory=CoarseningConfig)
    seed: int = 1

    def __post_init__(self):
        if self.n_tests < 2:
            raise ValueError("need at least two test vectors")
        if self.setup_cycles < 1:
            raise ValueError("setup_cycles must be at least 1")
        if self.inner_passes < 1:
            raise ValueError("inner_passes must be at least 1")


class Level:
    """One level (bootstrap.py:83-99).  Device operators are `d*`; the
    reference's attribute names materialise host scipy copies on access."""

    def __init__(self, index, B: DeviceCSR, d, M: DeviceCSR, N: DeviceCSR, split=None,
                 P: DeviceCSR | None = None, Q: DeviceCSR | None = None, geometry=None,
                 Bt: DeviceCSR | None = None, W: DeviceCSR | None = None):
        self.index = index
        self.dB, self.ddiag, self.dM, self.dN = B, d, M, N
        self.split = split
        self.dP, self.dQ, self.dBt, self.dW = P, Q, Bt, W
        self._geometry = geometry
        self._cache = {}

    def _h(self, key, M):
        if M is None:
            return None
        if key not in self._cache:
            self._cache[key] = M.to_host()
        return self._cache[key]

    @property
    def n(self) -> int:
        return self.dB.shape[0]

    @property
    def nnz(self) -> int:
        return self.dB.nnz

    B = property(lambda self: self._h("B", self.dB))
    M = property(lambda self: self._h("M", self.dM))
    N = property(lambda self: self._h("N", self.dN))
    P = property(lambda self: self._h("P", self.dP))
    Q = property(lambda self: self._h("Q", self.dQ))

    @property
    def diag(self) -> np.ndarray:
        return self.ddiag.cpu().numpy()

    @property
    def geometry(self):
        g = self._geometry
        if g is None:
            return None
        hc = g.host_coords if isinstance(g, AxisRanks) else g
        return hc.value() if hasattr(hc, "value") else hc


@dataclass
class Hierarchy:
    levels: list

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def finest(self) -> Level:
        return self.levels[0]

    @property
    def coarsest(self) -> Level:
        return self.levels[-1]


class SetupResult:
    """bootstrap.py:119-124; `x0` is materialised on the host on first access."""

    def __init__(self, hierarchy, triplets, dx0, seconds=0.0):
        self.hierarchy = hierarchy
        self.triplets = triplets
        self.dx0 = dx0
        self.seconds = seconds
        self._x0 = None

    @property
    def x0(self) -> np.ndarray:
        if self._x0 is None:
            self._x0 = self.dx0.cpu().numpy()
        return self._x0


def complexities(hierarchy: Hierarchy) -> tuple[float, float, int]:
    """Grid / operator complexity and depth (bootstrap.py:127-136)."""
    levels = hierarchy.levels
    if not levels:
        raise ValueError("empty hierarchy")
    n0 = levels[0].n
    nnz0 = max(levels[0].nnz, 1)
    return (float(sum(lv.n for lv in levels) / n0), float(sum(lv.nnz for lv in levels) / nnz0),
            len(levels))


def levels_at_least(hierarchy: Hierarchy, floor: int = 100) -> int:
    return sum(1 for lv in hierarchy.levels if lv.n >= floor)


class _SeedStream:
    """bootstrap.py:317-324."""

    def __init__(self, seed_sequence: np.random.SeedSequence):
        self._ss = seed_sequence

    def next(self) -> np.random.SeedSequence:
        return self._ss.spawn(1)[0]


class _LevelOps:
    """Device state of one level reused across the setup: B, B^T, diag, skip
    masks, adjacency (built lazily, once)."""

    def __init__(self, B: DeviceCSR, Bt: DeviceCSR | None = None):
        self.B = B
        self.Bt = Bt if Bt is not None else engine.transpose(B)
        self.d = engine.diag(B)
        self.skip = engine.degenerate_rows(B, self.d)
        self.skip_t = engine.degenerate_rows(self.Bt, self.d)
        self._adj = None

    @property
    def adj(self):
        if self._adj is None:
            self._adj = engine.sym_pattern(self.B, self.Bt)
        return self._adj


def _mass(M: DeviceCSR):
    """None for an identity mass (engine fast path, bit-identical)."""
    return None if M.is_identity else M


class _OwnedDraws(tuple):
    """(right, left) device blocks drawn by run_setup itself: relaxed in place, no defensive copy."""


def init_test_vectors(B, cfg: SetupConfig, rng=None, draws=None, ops: _LevelOps | None = None, comm=None):
    """Smoothed random left/right test vectors; left slot 0 constant (bootstrap.py:180-202).

    The raw draws come from `rng.standard_normal((r, n))` twice (right, then
    left) as in the reference, or from `draws=(right, left)` ((r, n) arrays,
    e.g. the BASELINE uniform(0,1) vectors).  They are host-generated inputs
    uploaded once; the smoothing, normalisation, sigmas and ordering run on
    device.
    """
    A = as_device(B)
    ops = ops or _LevelOps(A)
    n = A.shape[0]
    r = cfg.n_tests
    if isinstance(draws, str):
        if draws != "uniform":
            raise ValueError(f"unknown draws {draws!r} (expected 'uniform' or a (right, left) pair)")
        # BASELINE's uniform(0,1) vectors, default_rng(cfg.seed).random((r, n)) twice,
        # generated on the device (engine.uniform_draws: numpy's PCG64, bit-identical)
        right_h, left_h = engine.uniform_draws(cfg.seed, r, n)
    elif draws is None:
        if rng is None:
            rng = np.random.default_rng(np.random.SeedSequence(cfg.seed))
        right_h = rng.standard_normal((r, n))
        left_h = rng.standard_normal((r, n))
    else:
        right_h, left_h = draws
    if isinstance(right_h, torch.Tensor):
        # device-resident draws, already n x k interleaved; the smoothing works in place, so a
        # caller's blocks are copied and the ones drawn here are not
        own = isinstance(draws, (str, _OwnedDraws))
        V = right_h if own else right_h.clone()
        U = left_h if own else left_h.clone()
    else:
        V = engine.to_device_vec(np.ascontiguousarray(np.asarray(right_h, dtype=np.float64).T))
        U = engine.to_device_vec(np.ascontiguousarray(np.asarray(left_h, dtype=np.float64).T))
    sig = torch.zeros(r, dtype=torch.float64, device=device())
    sm = cfg.smoother
    # nu1 homogeneous sweeps per slot, no runaway rescaling (bootstrap.py:191-194)
    if _slot_partitioned(comm, n, r):
        _smooth_slots(ops, None, None, U, V, sig, cfg, 0, 2, comm)
    else:
        engine.smooth_block(A, ops.Bt, None, None, ops.d, ops.skip, ops.skip_t, U, V, sig,
                            sm.sweeps_pre, sm.omega, inhomogeneous=0, smooth=2, refresh=0)
    engine.col_fill(U, 0, 1.0 / np.sqrt(n))
    engine.normalize_cols(V)
    engine.normalize_cols(U)
    engine.refresh_sigmas(A, None, None, U, V, sig)
    s = sig.cpu().numpy()
    order = np.concatenate([[0], 1 + np.argsort(s[1:], kind="stable")])
    if not np.array_equal(order, np.arange(r)):
        U = engine.permute_cols(U, order)
        V = engine.permute_cols(V, order)
        sig = engine.to_device_vec(s[order])
    return TripletSet(sig, U, V)


def _band_min_n() -> int:
    import os
    return int(os.environ.get("BAMG_BAND_N", "2048"))


def coarsest_triplets(B, M, N, r: int, Bt: DeviceCSR | None = None, warm: "TripletSet | None" = None) -> TripletSet:
    """Exact generalized singular triplets of the coarsest operator (bootstrap.py:205-281).

    Large banded levels (the lattice chains keep the fine ordering, so the
    coarsest operators have half-bandwidth ~ side + 1) take the block-
    tridiagonal path (csrc/band.cu: no dense n x n matrix); everything else,
    or a band factorisation that is not certified, the dense path."""
    A, Md, Nd = as_device(B), as_device(M), as_device(N)
    n = A.shape[0]
    if n >= _band_min_n():
        out = engine.coarsest_triplets_band(A, Bt if Bt is not None else engine.transpose(A), Md, Nd, r,
                                            warm_right=warm.dright if warm is not None else None)
        if out is not None:
            U, V, s, lu = out
            trips = TripletSet(s, U, V)
            trips.coarse_pinv = lu
            return trips
    Bd = engine.csr_to_dense(A)
    Mdd = engine.csr_to_dense(Md)
    Ndd = engine.csr_to_dense(Nd)
    # the derived B^+ is one more dense n x n block alive next to B, M, N, K and
    # K^+ (5 x 18 GB at cfg3's n = 47,824): above 4 GB the V-cycle factorises
    # B itself after the setup's dense temporaries are gone
    U, V, s, Z = engine.coarsest_triplets(Bd, Mdd, Ndd, n, r, with_pinv=8 * n * n <= (4 << 30))
    # Z: B's explicit pseudo-inverse derived from the triplet factors, or the
    # kept bordered LU of B (engine.CoarseLU) when the implicit path ran
    trips = TripletSet(s, U, V)
    # B's pseudo-inverse from the same factors (large path): the V-cycle takes
    # it instead of factorising B again (solver.VCycleOperator)
    trips.coarse_pinv = Z
    return trips


#: levels below this many rows are smoothed replicated (the all-gather would cost more than it saves)
SLOT_PARTITION_MIN_ROWS = 1 << 14


def _slot_partitioned(comm, n: int, r: int) -> bool:
    return comm is not None and comm.world > 1 and r >= comm.world and n >= SLOT_PARTITION_MIN_ROWS


def _smooth_slots(ops: _LevelOps, M, N, U, V, sig, cfg: SetupConfig, inhomogeneous: int, smooth: int, comm):
    """The block's sweeps with the r triplet slots split over the ranks (multi-GPU setup).

    The coupled sweeps of bootstrap.py:291-308 never mix slots -- slot k's u, v and sigma only
    see each other -- so rank q relaxes slots [b_q, b_q+1) against the replicated operators
    with no communication at all, and ONE all-gather per side returns the full n x r blocks
    (NVLink / NVSwitch: 2 n r 8 bytes per level).  Every column goes through the same sweep
    arithmetic as on one GPU; only the in-sweep Rayleigh quotients' partial-sum grouping depends
    on the slice width, so the hierarchy's patterns are those of the single-GPU setup and its
    values agree to round-off."""
    from .distributed import slot_bounds
    r = U.shape[1]
    b = slot_bounds(r, comm.world)
    s0, s1 = int(b[comm.rank]), int(b[comm.rank + 1])
    Ul, Vl = U[:, s0:s1].contiguous(), V[:, s0:s1].contiguous()
    sl = sig[s0:s1].clone()
    sm = cfg.smoother
    engine.smooth_block(ops.B, ops.Bt, M, N, ops.d, ops.skip, ops.skip_t, Ul, Vl, sl,
                        sm.sweeps_pre, sm.omega, inhomogeneous, smooth=smooth, refresh=0)
    U.copy_(comm.all_gather_cols(Ul, b))
    V.copy_(comm.all_gather_cols(Vl, b))
    sig.copy_(comm.all_gather_cols(sl.reshape(1, -1), b).reshape(-1))


def _smooth_block(ops: _LevelOps, M, N, trips: TripletSet, cfg: SetupConfig, inhomogeneous: bool, comm=None):
    """bootstrap.py:284-314 in one engine call (slots split over the ranks of `comm`)."""
    sm = cfg.smoother
    if _slot_partitioned(comm, trips.n, trips.r):
        _smooth_slots(ops, _mass(M), _mass(N), trips.dleft, trips.dright, trips.dsigmas, cfg,
                      int(inhomogeneous), 1, comm)
        # normalise, pin the constant left slot, refresh the sigmas: replicated on the full block
        engine.smooth_block(ops.B, ops.Bt, _mass(M), _mass(N), ops.d, ops.skip, ops.skip_t,
                            trips.dleft, trips.dright, trips.dsigmas, 0, sm.omega, 0, smooth=0, refresh=1)
        return
    engine.smooth_block(ops.B, ops.Bt, _mass(M), _mass(N), ops.d, ops.skip, ops.skip_t,
                        trips.dleft, trips.dright, trips.dsigmas, sm.sweeps_pre, sm.omega,
                        int(inhomogeneous), smooth=1, refresh=1)


def _spgemm_many(products, comm=None):
    """engine.spgemm_many, the rows of every product split over the ranks of `comm`
    (multi-GPU setup): row i of A B only needs row i of A, so rank q multiplies its
    contiguous block of A's rows by the replicated B and the blocks are all-gathered --
    the same rows, bit for bit (per-row accumulation order included), as the full product."""
    from .interp import PARTITION_STATS, ROW_PARTITION_MIN_ROWS
    if comm is None or comm.world == 1 or min(A.shape[0] for A, _, _ in products) < ROW_PARTITION_MIN_ROWS:
        return engine.spgemm_many(products)
    from .distributed import RowPartition, row_slice
    parts = [RowPartition(A.shape[0], comm.world) for A, _, _ in products]
    local = engine.spgemm_many([(row_slice(A, *pt.range(comm.rank)), Bm, order)
                                for (A, Bm, order), pt in zip(products, parts)])
    PARTITION_STATS["products"] += len(products)
    return [comm.all_gather_csr_rows(Cl, pt) for Cl, pt in zip(local, parts)]


def _operator_degenerate(Bc: DeviceCSR) -> bool:
    """bootstrap.py:332-334."""
    d = engine.diag(Bc)
    bad = engine.count_nonpositive(d)
    if _DEBUG:
        print(f"[bamg] galerkin n_c={Bc.shape[0]} nnz={Bc.nnz} nonpositive_diag={bad} "
              f"limit={SICK_DIAG_FRACTION * Bc.shape[0]:.1f}", file=sys.stderr, flush=True)
    return bad > SICK_DIAG_FRACTION * Bc.shape[0]


def _coarsest_level(depth, A, ops, Md, Nd, ranks, trips: TripletSet) -> Level:
    lev = Level(depth, A, ops.d, Md, Nd, geometry=ranks, Bt=ops.Bt)
    lev.coarse_pinv = getattr(trips, "coarse_pinv", None)
    return lev


def bootstrap_cycle(B, M, N, trips: TripletSet, cfg: SetupConfig, geometry=None, depth: int = 0,
                    first_cycle: bool = True, seed_stream: _SeedStream | None = None,
                    ops: _LevelOps | None = None, comm=None):
    """One recursive setup pass (bootstrap.py:337-392); returns (levels, triplets)."""
    A = as_device(B)
    if ops is None:
        with _phase("level_ops", depth):
            ops = _LevelOps(A)
    Md, Nd = as_device(M), as_device(N)
    n = A.shape[0]
    if seed_stream is None:
        seed_stream = _SeedStream(np.random.SeedSequence(cfg.seed))
    ranks = geometry
    if geometry is not None and not isinstance(geometry, AxisRanks):
        ranks = AxisRanks.from_geometry(geometry)

    split = None
    if n >= cfg.coarsening.stop_size and depth + 1 < cfg.coarsening.max_levels:
        seed = seed_stream.next()
        with _phase("split", depth):
            if cfg.coarsening.mode == "cr":
                split = make_splitting(A, ranks, cfg.coarsening, seed, adj=ops.adj, diag=ops.d)
            else:
                split = make_splitting(A, ranks, cfg.coarsening, seed)
        if _DEBUG:
            print(f"[bamg] level {depth} n={n} split n_c={split.n_coarse}", file=sys.stderr, flush=True)
        if split.n_coarse >= 0.9 * n or split.n_coarse == n:
            split = None  # coarsening stalled
    if split is None:
        if _DEBUG:
            print(f"[bamg] coarsest level {depth} n={n}", file=sys.stderr, flush=True)
        with _phase("coarsest", depth):
            trips = coarsest_triplets(A, Md, Nd, trips.r, Bt=ops.Bt, warm=trips)
        return [_coarsest_level(depth, A, ops, Md, Nd, ranks, trips)], trips

    with _phase("smooth", depth):
        _smooth_block(ops, Md, Nd, trips, cfg, inhomogeneous=not first_cycle, comm=comm)

    levels = None
    for _ in range(cfg.inner_passes):
        with _phase("weights", depth):
            v_tests = singular_test_weights(A, trips.dright)
            u_tests = singular_test_weights(A, trips.dleft, transpose_side=True,
                                            infinite_slot=0 if cfg.interp.constrain_constant_in_q else None,
                                            Bt=ops.Bt)
        with _phase("adjacency", depth):
            adj = ops.adj
        with _phase("ls_fit", depth):
            P, W = build_transfer_pair(A, split, v_tests, u_tests, cfg.interp, adj=adj, comm=comm)
        with _phase("galerkin", depth):
            # B_c = (Q B) P (sparse.py:102-117), M_c = Q M Q^T, N_c = P^T N P
            # (bootstrap.py:372-373): the independent products of each stage
            # are counted together (one host read per stage).  Identity masses
            # (the finest level): scipy's Q@I / I@P store every row reversed,
            # so (Q I) W and P^T (I P) are the products with Q's / P's rows
            # walked in reverse -- bit-identical, no identity product.
            Q = engine.transpose(W)
            Pt = engine.transpose(P)
            stage1 = [(Q, A, 1)]
            stage1.append((Q, W, engine.SPGEMM_REV_A) if Md.is_identity else (Q, Md, 1))
            stage1.append((Pt, P, engine.SPGEMM_REV_B) if Nd.is_identity else (Nd, P, 1))
            QB, QM, NP = _spgemm_many(stage1, comm)
            stage2 = [(QB, P, 0)]
            if not Md.is_identity:
                stage2.append((QM, W, 0))
            if not Nd.is_identity:
                stage2.append((Pt, NP, 0))
            out2 = _spgemm_many(stage2, comm)
            Bc = out2[0]
            Mc = QM if Md.is_identity else out2[1]
            Nc = NP if Nd.is_identity else out2[-1]
            sick = _operator_degenerate(Bc)
        if sick:
            if _DEBUG:
                print(f"[bamg] truncated at level {depth} n={n} (sick Galerkin product)", file=sys.stderr, flush=True)
            with _phase("coarsest", depth):
                trips = coarsest_triplets(A, Md, Nd, trips.r, Bt=ops.Bt, warm=trips)
            return [_coarsest_level(depth, A, ops, Md, Nd, ranks, trips)], trips
        with _phase("inject", depth):
            cranks = ranks.restrict(split) if ranks is not None else None
            cl = engine.gather_rows(trips.dleft, split.dcoarse)
            cr = engine.gather_rows(trips.dright, split.dcoarse)
            engine.normalize_cols(cl)
            engine.normalize_cols(cr)
        coarse = TripletSet(trips.dsigmas.clone(), cl, cr)
        sub_levels, coarse = bootstrap_cycle(Bc, Mc, Nc, coarse, cfg, cranks, depth + 1,
                                             first_cycle, seed_stream, comm=comm)
        # prolong: u <- Q^T u_c (= W u_c), v <- P v_c; normalise; pin; refresh; smooth
        with _phase("prolong", depth):
            U = engine.spmm(W, coarse.dleft)
            V = engine.spmm(P, coarse.dright)
            trips = TripletSet(coarse.dsigmas.clone(), U, V)
            engine.smooth_block(ops.B, ops.Bt, _mass(Md), _mass(Nd), ops.d, ops.skip, ops.skip_t,
                                U, V, trips.dsigmas, 0, cfg.smoother.omega, 0, smooth=0, refresh=1)
        with _phase("smooth", depth):
            _smooth_block(ops, Md, Nd, trips, cfg, inhomogeneous=True, comm=comm)
        levels = [Level(depth, A, ops.d, Md, Nd, split, P, Q, ranks, Bt=ops.Bt, W=W)] + sub_levels
    return levels, trips


def run_setup(problem, cfg: SetupConfig, draws=None, B_device: DeviceCSR | None = None, comm=None) -> SetupResult:
    """Full setup: initial vectors, the configured cycles, x0 (bootstrap.py:395-429).

    `draws=(right, left)` injects the raw (k, n) initial vectors (BASELINE's
    uniform(0,1) seed-0 vectors); `draws="uniform"` draws those vectors
    (default_rng(cfg.seed).random, right then left) on the device; otherwise
    the reference's own SeedSequence(seed).spawn(2)[0] standard-normal stream
    is used.

    `comm` (distributed.Comm of an initialised process group, one rank per GPU):
    the bootstrap relaxation -- the largest setup phase -- is split by triplet
    slot over the ranks (`_smooth_slots`); every rank ends with the same hierarchy.
    """
    t0 = time.perf_counter()
    A = B_device if B_device is not None else as_device(problem.B)
    n = A.shape[0]
    root = np.random.SeedSequence(cfg.seed)
    ss_init, ss_levels = root.spawn(2)
    if isinstance(draws, str) and draws == "uniform":
        # the seeded draws need nothing of the operator: generated first, so they overlap an
        # operator still being copied in (ChainProblem.B_ready)
        with _phase("draws"):
            draws = _OwnedDraws(engine.uniform_draws(cfg.seed, cfg.n_tests, n))
    ready = getattr(problem, "B_ready", None)
    if ready is not None:  # the operator's arrays were copied in on a side stream
        torch.cuda.current_stream().wait_event(ready)
    with _phase("level_ops"):
        # the generators' B = I - A has a handful of distinct values: the k = 1
        # sweeps / residuals / SpMVs of the solve stream its packed copy
        # (4 instead of 12 bytes per entry, same bits); redone every setup, on a
        # wrapper of its own so the hierarchy owns the packed arrays (the
        # caller's operator is left as it came)
        A = DeviceCSR(A.rowptr, A.col, A.val, A.shape, is_identity=A.is_identity)
        engine.pack_operator(A)
        ops = _LevelOps(A)
        if A.ptiles is not None:
            # a lattice chain: B^T has an interior stencil too (the k-wide sweeps of the left vectors)
            engine.attach_stencil(ops.Bt)
    rng = np.random.default_rng(ss_init) if draws is None else None
    with _phase("init"):
        trips = init_test_vectors(A, cfg, rng=rng, draws=draws, ops=ops, comm=comm)
    stream = _SeedStream(ss_levels)
    eye = DeviceCSR.identity(n)
    geometry = problem.geometry
    if geometry is not None and not isinstance(geometry, AxisRanks):
        ready = getattr(problem, "geometry_ready", None)
        if ready is not None:  # the coordinates were copied in on a side stream
            torch.cuda.current_stream().wait_event(ready)
        with _phase("axis_ranks"):
            geometry = AxisRanks.from_geometry(geometry)
    hierarchy = None
    for cycle in range(cfg.setup_cycles):
        levels, trips = bootstrap_cycle(A, eye, eye, trips, cfg, geometry=geometry, depth=0,
                                        first_cycle=(cycle == 0), seed_stream=stream, ops=ops, comm=comm)
        hierarchy = Hierarchy(levels)
        engine.col_fill(trips.dleft, 0, 1.0 / np.sqrt(n))
        engine.refresh_sigmas(A, None, None, trips.dleft, trips.dright, trips.dsigmas)
    dx0 = engine.sign_fix_l1(trips.dright, stride=trips.r, uniform_fallback=True)
    torch.cuda.synchronize()
    seconds = time.perf_counter() - t0
    return SetupResult(hierarchy, trips, dx0, seconds=seconds)


def triplet_residual(trips: TripletSet, B, M=None, N=None) -> float:
    """Setup progress metric (bootstrap.py:432-444), device reductions."""
    A = as_device(B)
    n = A.shape[0]
    Md = as_device(M) if M is not None else DeviceCSR.identity(n)
    Nd = as_device(N) if N is not None else DeviceCSR.identity(n)
    At = engine.transpose(A)
    s = trips.dsigmas
    Bv = engine.spmm(A, trips.dright)
    Mu = engine.spmm(Md, trips.dleft)
    Btu = engine.spmm(At, trips.dleft)
    Nv = engine.spmm(Nd, trips.dright)
    r1 = engine.col_norms(Bv - s * Mu)
    r2 = engine.col_norms(Btu - s * Nv)
    return float((r1 + r2).sum().item())


def export_hierarchy(hierarchy: Hierarchy, directory) -> None:
    """Matrix Market per level + JSON manifest (bootstrap.py:447-469)."""
    from pathlib import Path

    from scipy.io import mmwrite
    from scipy import sparse as sp

    out = Path(directory)
    out.mkdir(parents=True, exist_ok=True)
    o_g, o_c, depth = complexities(hierarchy)
    manifest = {"levels": [], "grid_complexity": o_g, "operator_complexity": o_c, "depth": depth}

    def save(path, M):
        mmwrite(str(path), sp.coo_matrix(M), comment="", field="real", precision=17,
                symmetry="general")

    for lev in hierarchy.levels:
        entry = {"index": lev.index, "n": int(lev.n), "nnz": int(lev.nnz)}
        save(out / f"B_{lev.index}.mtx", lev.B)
        if lev.dP is not None:
            save(out / f"P_{lev.index}.mtx", lev.P)
            save(out / f"Q_{lev.index}.mtx", lev.Q)
            split_file = f"splitting_{lev.index}.json"
            (out / split_file).write_text(lev.split.to_json())
            entry["splitting"] = split_file
            entry["n_coarse"] = int(lev.split.n_coarse)
        manifest["levels"].append(entry)
    (out / "hierarchy.json").write_text(json.dumps(manifest, indent=2, sort_keys=True))
