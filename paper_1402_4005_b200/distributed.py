"""Row-partitioned solve phase across ranks.

One process per GPU.  Every level of the hierarchy above the agglomeration
threshold is split into contiguous row blocks (tandem / uniform lattices are
ordered by strips, so a block is a strip and its halo is one grid row); each
rank keeps its rows of B_l, Q_l (coarse rows) and P_l (fine rows) with columns
renumbered into a halo-extended local numbering: owned columns first, then the
halo ordered by owner rank.  Per application:

  * SpMV / Jacobi sweep / residual: pack the entries peers need
    (bamg_gather_rows), one grouped NCCL send/recv per neighbour
    (torch.distributed.batch_isend_irecv; host-staged when the backend is
    gloo), then the bit-exact CSR-stream kernel on the local rows;
  * GMRES: CGS2 with rank-local fused dot / update passes (bamg_mdot,
    bamg_mupdate) and one all-reduce per pass, the Hessenberg bookkeeping
    replicated on every rank from the all-reduced scalars;
  * agglomeration: at the first level with fewer than `agglomerate_rows` rows
    the right-hand side is all-gathered and the remaining levels run
    replicated on every rank (the single-GPU VCycleOperator), each rank keeping
    its slice of the correction.

Row-local kernels make the result independent of the rank count up to the
order of the all-reduced sums.  The plan construction (which rows each rank
needs from which peer) renumbers the rank's slice of each DEVICE operator on
the device; only the halo id lists cross to the host (for the all-gather of
requests).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist
from scipy import sparse as sp

from . import _lib, engine
from .device import DeviceCSR, device


# ---------------------------------------------------------------- partition
class RowPartition:
    """Contiguous, balanced row blocks: rank r owns [offsets[r], offsets[r+1])."""

    def __init__(self, n: int, world: int):
        self.n = int(n)
        self.world = int(world)
        base, extra = divmod(self.n, self.world)
        sizes = np.array([base + (1 if r < extra else 0) for r in range(self.world)], dtype=np.int64)
        self.offsets = np.concatenate([[0], np.cumsum(sizes)])

    def range(self, rank: int):
        return int(self.offsets[rank]), int(self.offsets[rank + 1])

    def owner(self, idx):
        return np.searchsorted(self.offsets, np.asarray(idx), side="right") - 1


def slot_bounds(k: int, world: int) -> np.ndarray:
    """Test-vector slots [b[r], b[r+1]) smoothed by rank r (as even as k allows)."""
    return np.array([(k * r) // world for r in range(world + 1)], dtype=np.int64)


def row_slice(A, r0: int, r1: int):
    """Rows [r0, r1) of a DeviceCSR as a DeviceCSR over views of its arrays (one host read)."""
    from .device import DeviceCSR
    ends = A.rowptr[[r0, r1]].cpu()
    j0, j1 = int(ends[0]), int(ends[1])
    rp = (A.rowptr[r0:r1 + 1] - j0).contiguous()
    return DeviceCSR(rp, A.col[j0:j1], A.val[j0:j1], (r1 - r0, A.shape[1]))


@dataclass
class HaloPlan:
    """Exchange plan of one local operator's halo-extended numbering."""

    n_own: int
    halo_ids: np.ndarray          # global column ids of the halo, ordered by owner
    recv_counts: dict             # peer -> number of halo entries received
    recv_offset: dict             # peer -> offset into the halo segment
    send_local: dict              # peer -> int32 local row indices to send (numpy)


class Comm:
    """torch.distributed wrapper: NCCL p2p on device buffers, host staging for gloo."""

    def __init__(self):
        self.active = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if self.active else 0
        self.world = dist.get_world_size() if self.active else 1
        self.gloo = self.active and dist.get_backend() == "gloo"

    def all_gather_object(self, obj):
        if not self.active:
            return [obj]
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def allreduce_(self, t: torch.Tensor):
        if not self.active or self.world == 1:
            return t
        if self.gloo:
            h = t.cpu()
            dist.all_reduce(h)
            t.copy_(h)
        else:
            dist.all_reduce(t)
        return t

    def all_gather_vec(self, own: torch.Tensor, part: RowPartition) -> torch.Tensor:
        """Full vector from every rank's block (rank order)."""
        if not self.active or self.world == 1:
            return own.clone()
        sizes = [int(part.offsets[r + 1] - part.offsets[r]) for r in range(self.world)]
        mx = max(sizes)
        pad = torch.zeros(mx, dtype=own.dtype, device=own.device)
        pad[: own.numel()] = own
        if self.gloo:
            hp = pad.cpu()
            bufs = [torch.empty_like(hp) for _ in range(self.world)]
            dist.all_gather(bufs, hp)
            bufs = [b.to(own.device) for b in bufs]
        else:
            bufs = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(bufs, pad)
        return torch.cat([bufs[r][: sizes[r]] for r in range(self.world)])

    def all_gather_cols(self, own: torch.Tensor, bounds) -> torch.Tensor:
        """n x k block from every rank's n x (bounds[r+1] - bounds[r]) column slice."""
        if not self.active or self.world == 1:
            return own
        n = own.shape[0]
        widths = [int(bounds[r + 1] - bounds[r]) for r in range(self.world)]
        mx = max(widths)
        pad = own if own.shape[1] == mx else torch.cat(
            [own, torch.zeros((n, mx - own.shape[1]), dtype=own.dtype, device=own.device)], dim=1)
        pad = pad.contiguous()
        if self.gloo:
            hp = pad.cpu()
            bufs = [torch.empty_like(hp) for _ in range(self.world)]
            dist.all_gather(bufs, hp)
            bufs = [b.to(own.device) for b in bufs]
        else:
            bufs = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(bufs, pad)
        return torch.cat([bufs[r][:, : widths[r]] for r in range(self.world)], dim=1).contiguous()

    def all_gather_flat(self, own: torch.Tensor, sizes=None) -> torch.Tensor:
        """Concatenation (rank order) of every rank's 1-D tensor; `sizes` = their lengths when
        every rank already knows them (saves the size all-gather)."""
        if not self.active or self.world == 1:
            return own
        if sizes is None:
            sizes = self.all_gather_object(int(own.numel()))
        mx = max(max(sizes), 1)
        pad = torch.zeros(mx, dtype=own.dtype, device=own.device)
        pad[: own.numel()] = own
        if self.gloo:
            hp = pad.cpu()
            bufs = [torch.empty_like(hp) for _ in range(self.world)]
            dist.all_gather(bufs, hp)
            bufs = [b.to(own.device) for b in bufs]
        else:
            bufs = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(bufs, pad)
        return torch.cat([bufs[r][: sizes[r]] for r in range(self.world)])

    def all_gather_csr_rows(self, C_own, part: "RowPartition"):
        """Full CSR from every rank's block of rows (rank order): per-row counts, columns and
        values are concatenated, the row pointer is their running sum (int32, as everywhere)."""
        from .device import DeviceCSR
        if not self.active or self.world == 1:
            return C_own
        rows = [int(part.offsets[r + 1] - part.offsets[r]) for r in range(self.world)]
        counts = self.all_gather_flat((C_own.rowptr[1:] - C_own.rowptr[:-1]).contiguous(), rows)
        nnzs = self.all_gather_object(int(C_own.nnz))
        col = self.all_gather_flat(C_own.col[: C_own.nnz].contiguous(), nnzs)
        val = self.all_gather_flat(C_own.val[: C_own.nnz].contiguous(), nnzs)
        rp = torch.zeros(part.n + 1, dtype=torch.int32, device=counts.device)
        rp[1:] = torch.cumsum(counts, 0, dtype=torch.int32)
        return DeviceCSR(rp, col, val, (part.n, C_own.shape[1]))

    def exchange(self, x_ext: torch.Tensor, plan: HaloPlan, sendbufs: dict, sendidx: dict):
        """Fill x_ext[n_own:] with the halo values owned by the peers."""
        if not plan.recv_counts and not plan.send_local:
            return
        # pack what the peers need from our owned block (device index lists)
        for peer, idx in sendidx.items():
            _lib.call("bamg_gather_rows", _lib.ptr(x_ext), _lib.ptr(idx), idx.numel(), 1,
                      _lib.ptr(sendbufs[peer]))
        ops = []
        if self.gloo:
            torch.cuda.synchronize()
            staged = {}
            for peer in sorted(set(plan.send_local) | set(plan.recv_counts)):
                if peer in plan.send_local:
                    ops.append(dist.P2POp(dist.isend, sendbufs[peer].cpu(), peer))
                if peer in plan.recv_counts:
                    staged[peer] = torch.empty(plan.recv_counts[peer], dtype=torch.float64)
                    ops.append(dist.P2POp(dist.irecv, staged[peer], peer))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            for peer, h in staged.items():
                o = plan.n_own + plan.recv_offset[peer]
                x_ext[o:o + h.numel()].copy_(h.to(x_ext.device))
            return
        for peer in sorted(set(plan.send_local) | set(plan.recv_counts)):
            if peer in plan.send_local:
                ops.append(dist.P2POp(dist.isend, sendbufs[peer], peer))
            if peer in plan.recv_counts:
                o = plan.n_own + plan.recv_offset[peer]
                ops.append(dist.P2POp(dist.irecv, x_ext[o:o + plan.recv_counts[peer]], peer))
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def build_plan(needed_global: np.ndarray, col_part: RowPartition, rank: int, comm: Comm):
    """Halo order and send lists for the global columns this rank needs off-rank."""
    c0, c1 = col_part.range(rank)
    halo = np.unique(needed_global[(needed_global < c0) | (needed_global >= c1)])
    owners = col_part.owner(halo)
    order = np.lexsort((halo, owners))
    halo, owners = halo[order], owners[order]
    recv_counts, recv_offset = {}, {}
    requests = {}
    off = 0
    for peer in np.unique(owners):
        ids = halo[owners == peer]
        recv_counts[int(peer)] = int(ids.size)
        recv_offset[int(peer)] = off
        requests[int(peer)] = ids
        off += ids.size
    everyone = comm.all_gather_object(requests)
    send_local = {}
    for peer, req in enumerate(everyone):
        if peer == rank or rank not in req:
            continue
        send_local[peer] = (np.asarray(req[rank]) - c0).astype(np.int32)
    return HaloPlan(c1 - c0, halo, recv_counts, recv_offset, send_local)


def localize_host(A: sp.csr_array, row_part: RowPartition, col_part: RowPartition, rank: int, comm: Comm):
    """Rank-local rows of A with halo-extended column numbering + exchange plan
    (host arrays: indptr, local columns, values, extended width, plan)."""
    r0, r1 = row_part.range(rank)
    loc = sp.csr_array(A[r0:r1])
    cols = loc.indices.astype(np.int64)
    plan = build_plan(cols, col_part, rank, comm)
    c0, c1 = col_part.range(rank)
    own = (cols >= c0) & (cols < c1)
    new = np.empty_like(cols)
    new[own] = cols[own] - c0
    if plan.halo_ids.size:
        pos = np.searchsorted(np.sort(plan.halo_ids), cols[~own])
        sorted_ids = np.sort(plan.halo_ids)
        # position in the owner-ordered halo
        rank_of_sorted = np.empty(plan.halo_ids.size, dtype=np.int64)
        rank_of_sorted[np.argsort(plan.halo_ids)] = np.arange(plan.halo_ids.size)
        assert np.array_equal(sorted_ids[pos], cols[~own])
        new[~own] = plan.n_own + rank_of_sorted[pos]
    n_ext = plan.n_own + plan.halo_ids.size
    # storage order keeps the global ascending column order, so each row's
    # sequential sum is the single-GPU (and scipy) order
    return loc.indptr.astype(np.int32), new.astype(np.int32), np.ascontiguousarray(loc.data), n_ext, plan


def _plan_from_halo(halo_ids: np.ndarray, col_part: RowPartition, rank: int, comm: Comm) -> HaloPlan:
    """Exchange plan for an owner-ordered halo (ids ascending within each owner)."""
    c0, c1 = col_part.range(rank)
    owners = col_part.owner(halo_ids)
    recv_counts, recv_offset, requests = {}, {}, {}
    off = 0
    for peer in np.unique(owners):
        ids = halo_ids[owners == peer]
        recv_counts[int(peer)] = int(ids.size)
        recv_offset[int(peer)] = off
        requests[int(peer)] = ids
        off += ids.size
    everyone = comm.all_gather_object(requests)
    send_local = {}
    for peer, req in enumerate(everyone):
        if peer == rank or rank not in req:
            continue
        send_local[peer] = (np.asarray(req[rank]) - c0).astype(np.int32)
    return HaloPlan(c1 - c0, halo_ids, recv_counts, recv_offset, send_local)


def localize_device(A: DeviceCSR, row_part: RowPartition, col_part: RowPartition, rank: int, comm: Comm):
    """localize_host on the device operator: the rank's row slice stays in HBM,
    its columns are renumbered on the device (owned first, then the halo in
    owner order -- a contiguous partition makes ascending ids owner-ordered),
    and only the halo ids (a few grid rows for the lattice strips) come to the
    host for the plan.  No copy of the operator leaves the device."""
    r0, r1 = row_part.range(rank)
    c0, c1 = col_part.range(rank)
    rp = A.rowptr[r0:r1 + 1]
    e0, e1 = (int(v) for v in rp[[0, -1]].tolist())
    cols = A.col[e0:e1].long()
    vals = A.val[e0:e1]
    own = (cols >= c0) & (cols < c1)
    halo = torch.unique(cols[~own])
    new = torch.empty_like(cols)
    new[own] = cols[own] - c0
    new[~own] = (c1 - c0) + torch.searchsorted(halo, cols[~own])
    plan = _plan_from_halo(halo.cpu().numpy().astype(np.int64), col_part, rank, comm)
    n_ext = plan.n_own + int(halo.numel())
    M = DeviceCSR((rp - e0).to(torch.int32).contiguous(), new.to(torch.int32).contiguous(), vals.contiguous(),
                  (r1 - r0, n_ext))
    return M, plan


def localize(A, row_part: RowPartition, col_part: RowPartition, rank: int, comm: Comm):
    """Rank-local operator + plan: device path for a DeviceCSR, host path for scipy."""
    if isinstance(A, DeviceCSR):
        return localize_device(A, row_part, col_part, rank, comm)
    indptr, cols, vals, n_ext, plan = localize_host(A, row_part, col_part, rank, comm)
    M = DeviceCSR(torch.from_numpy(indptr).to(device()), torch.from_numpy(cols).to(device()),
                  torch.from_numpy(vals).to(device()), (indptr.size - 1, n_ext))
    return M, plan


class _DistOp:
    def __init__(self, A, row_part, col_part, rank, comm):
        self.M, self.plan = localize(A, row_part, col_part, rank, comm)
        self.sendidx = {p: torch.from_numpy(idx).to(device()) for p, idx in self.plan.send_local.items()}
        self.sendbufs = {p: torch.empty(idx.size, dtype=torch.float64, device=device())
                         for p, idx in self.plan.send_local.items()}
        self.comm = comm

    @property
    def n_ext(self):
        return self.M.shape[1]

    def halo(self, x_ext):
        self.comm.exchange(x_ext, self.plan, self.sendbufs, self.sendidx)


class DistLevel:
    def __init__(self, lev, part, cpart, rank, comm, omega):
        self.part, self.cpart = part, cpart
        self.r0, self.r1 = part.range(rank)
        self.n_own = self.r1 - self.r0
        self.B = _DistOp(lev.dB, part, part, rank, comm)
        d = lev.ddiag[self.r0:self.r1].contiguous()
        self.d = d
        self.skip = engine.degenerate_rows(lev.dB, lev.ddiag)[self.r0:self.r1].contiguous()
        self.omega = omega
        if cpart is not None:
            c0, c1 = cpart.range(rank)
            self.Q = _DistOp(lev.dQ, cpart, part, rank, comm)   # coarse rows, fine columns
            self.P = _DistOp(lev.dP, part, cpart, rank, comm)   # fine rows, coarse columns
            self.r_ext = torch.empty(self.Q.n_ext, dtype=torch.float64, device=device())
            self.xc_ext = torch.empty(self.P.n_ext, dtype=torch.float64, device=device())
        ne = self.B.n_ext
        self.x = [torch.empty(ne, dtype=torch.float64, device=device()) for _ in range(2)]
        self.b = torch.empty(self.n_own, dtype=torch.float64, device=device())


class DistVCycle:
    """The V-cycle of a (replicated) Hierarchy applied to row-partitioned vectors."""

    def __init__(self, hierarchy, smoother, comm: Comm | None = None, agglomerate_rows: int = 1 << 16,
                 coarsest_rank_tol: float = 1e-12):
        from .bootstrap import Hierarchy
        from .solver import VCycleOperator
        self.comm = comm or Comm()
        self.sm = smoother
        rank, world = self.comm.rank, self.comm.world
        levels = hierarchy.levels
        L = len(levels)
        agg = L - 1
        for i, lv in enumerate(levels):
            if lv.n < agglomerate_rows or i == L - 1:
                agg = i
                break
        self.agg = agg
        parts = [RowPartition(lv.n, world) for lv in levels]
        self.parts = parts
        self.levels = [DistLevel(levels[i], parts[i], parts[i + 1], rank, self.comm, smoother.omega)
                       for i in range(agg)]
        self.tail = VCycleOperator(Hierarchy(levels[agg:]), smoother, coarsest_rank_tol)
        self.n_own = parts[0].range(rank)[1] - parts[0].range(rank)[0]

    def _tail(self, b_own, part):
        full = self.comm.all_gather_vec(b_own, part)
        x_full = self.tail.apply(full)
        r0, r1 = part.range(self.comm.rank)
        return x_full[r0:r1].contiguous()

    def apply(self, b_own: torch.Tensor) -> torch.Tensor:
        if self.agg == 0:
            return self._tail(b_own, self.parts[0])
        return self._down(0, b_own)

    def _down(self, l, b_own):
        lv = self.levels[l]
        sm = self.sm
        om = float(sm.omega)
        cur, oth = lv.x[0], lv.x[1]
        if sm.sweeps_pre > 0:
            _lib.call("bamg_jacobi_zero", lv.n_own, _lib.ptr(b_own), _lib.ptr(lv.d), _lib.ptr(lv.skip), om,
                      _lib.ptr(cur))
            for _ in range(sm.sweeps_pre - 1):
                lv.B.halo(cur)
                _lib.call("bamg_jacobi", lv.B.M.ref(), _lib.ptr(lv.d), _lib.ptr(lv.skip), _lib.ptr(b_own), None,
                          _lib.ptr(cur), _lib.ptr(oth), 1, om, None)
                cur, oth = oth, cur
        else:
            cur.zero_()
        lv.B.halo(cur)
        _lib.call("bamg_residual", lv.B.M.ref(), _lib.ptr(b_own), _lib.ptr(cur), _lib.ptr(lv.r_ext))
        lv.Q.halo(lv.r_ext)
        bc = torch.empty(lv.Q.M.shape[0], dtype=torch.float64, device=device())
        _lib.call("bamg_spmv", lv.Q.M.ref(), _lib.ptr(lv.r_ext), _lib.ptr(bc))
        if l + 1 == len(self.levels):
            xc = self._tail(bc, self.parts[l + 1])
        else:
            xc = self._down(l + 1, bc)
        nco = xc.numel()
        lv.xc_ext[:nco].copy_(xc)
        lv.P.halo(lv.xc_ext)
        _lib.call("bamg_addmv", lv.P.M.ref(), _lib.ptr(lv.xc_ext), _lib.ptr(cur), _lib.ptr(oth))
        cur, oth = oth, cur
        for _ in range(sm.sweeps_post):
            lv.B.halo(cur)
            _lib.call("bamg_jacobi", lv.B.M.ref(), _lib.ptr(lv.d), _lib.ptr(lv.skip), _lib.ptr(b_own), None,
                      _lib.ptr(cur), _lib.ptr(oth), 1, om, None)
            cur, oth = oth, cur
        return cur[: lv.n_own].clone()


def _lincomb(vecs, coefs, base=None):
    """base + sum_i coefs_i vecs_i with the engine's fused combine kernel."""
    n = vecs[0].numel() if vecs else base.numel()
    out = torch.empty(n, dtype=torch.float64, device=device())
    table = torch.tensor([v.data_ptr() for v in vecs] or [0], dtype=torch.int64, device=device())
    cf = torch.tensor(list(coefs) or [0.0], dtype=torch.float64, device=device())
    _lib.call("bamg_combine", _lib.ptr(table), len(vecs), _lib.ptr(cf), _lib.ptr(base), None, n, _lib.ptr(out))
    return out


class DistSolver:
    """Row-partitioned left-preconditioned GMRES (solver.py:136-226 semantics, CGS2)."""

    def __init__(self, hierarchy, smoother, comm: Comm | None = None, agglomerate_rows: int = 1 << 16):
        self.comm = comm or Comm()
        self.vc = DistVCycle(hierarchy, smoother, self.comm, agglomerate_rows)
        lev0 = hierarchy.levels[0]
        self.part = RowPartition(lev0.n, self.comm.world)
        self.r0, self.r1 = self.part.range(self.comm.rank)
        self.B = _DistOp(lev0.dB, self.part, self.part, self.comm.rank, self.comm)
        self.x_ext = torch.empty(self.B.n_ext, dtype=torch.float64, device=device())
        self.n_own = self.r1 - self.r0

    def spmv(self, v_own):
        self.x_ext[: self.n_own].copy_(v_own)
        self.B.halo(self.x_ext)
        y = torch.empty(self.n_own, dtype=torch.float64, device=device())
        _lib.call("bamg_spmv", self.B.M.ref(), _lib.ptr(self.x_ext), _lib.ptr(y))
        return y

    def _dots(self, vecs, w):
        m = len(vecs)
        table = torch.tensor([v.data_ptr() for v in vecs], dtype=torch.int64, device=device())
        out = torch.empty(m, dtype=torch.float64, device=device())
        _lib.call("bamg_mdot", _lib.ptr(table), m, _lib.ptr(w), self.n_own, _lib.ptr(out))
        self.comm.allreduce_(out)
        return table, out

    def _norm2(self, v):
        out = torch.empty(1, dtype=torch.float64, device=device())
        _lib.call("bamg_col_dots", _lib.ptr(v), _lib.ptr(v), self.n_own, 1, _lib.ptr(out))
        self.comm.allreduce_(out)
        return float(out.item())

    def op(self, v):
        return self.vc.apply(self.spmv(v))

    def metric(self, x):
        nx = np.sqrt(self._norm2(x))
        if nx == 0.0:
            return np.inf
        return np.sqrt(self._norm2(self.spmv(x))) / nx

    #: basis vectors the fused passes keep in registers (csrc/solver.cu CGS_MAXM)
    MAX_FUSED = 64

    def _table(self, vecs):
        return torch.tensor([v.data_ptr() for v in vecs], dtype=torch.int64, device=device())

    def _bx_norm2_local(self, x):
        y = self.spmv(x)
        out = torch.empty(1, dtype=torch.float64, device=device())
        _lib.call("bamg_col_dots", _lib.ptr(y), _lib.ptr(y), self.n_own, 1, _lib.ptr(out))
        return out

    def solve(self, x0_own, restart=None, max_iters=1000, rtol=1e-8):
        """The engine's Arnoldi step (csrc/solver.cu, two-pass CGS2 through the Gram
        matrix) on this rank's rows: pass A (V^T w, |w|^2) -> ONE all-reduce -> the
        coefficients c = 2 h1 - G h1, the new vector's norm and the Givens update on the
        host (the scalars the stopping test reads anyway) -> pass B (v_new, x, V^T v_new,
        |x|^2) and |Bx|^2 -> ONE all-reduce.  Two reads of the local basis block, two
        all-reduces and two host reads per iteration (the first version took five
        all-reduces and four basis sweeps).  Cycles longer than 64 vectors are restarted
        at 64 (the fused passes hold the row's basis values in registers)."""
        from scipy.linalg import solve_triangular
        x0 = x0_own.clone()
        rhs = self.vc.apply(_lincomb([self.spmv(x0)], [-1.0]))  # C(b - B x0), b = 0
        hist = [self.metric(x0)]
        if hist[0] <= rtol:
            return 0, hist, True, x0
        dev = device()
        e = torch.zeros_like(x0)
        x = x0.clone()
        its, done = 0, False
        while its < max_iters and not done:
            r = _lincomb([self.op(e)], [-1.0], base=rhs) if its else rhs.clone()
            beta = np.sqrt(self._norm2(r))
            if beta == 0.0:
                break
            m = min(restart or max_iters, max_iters - its, self.MAX_FUSED)
            V = [_lincomb([r], [1.0 / beta])]
            G = np.zeros((m + 1, m + 1))
            G[0, 0] = 1.0
            R = np.zeros((m, m))
            g = np.zeros(m + 1)
            g[0] = beta
            cs, sn = np.zeros(m), np.zeros(m)
            used, happy = 0, False
            e_try = e
            for j in range(m):
                mj = j + 1
                w = self.op(V[j])
                table = self._table(V)
                out1 = torch.empty(mj + 1, dtype=torch.float64, device=dev)
                _lib.call("bamg_cgs_dots", _lib.ptr(table), mj, _lib.ptr(w), self.n_own, _lib.ptr(out1))
                self.comm.allreduce_(out1)
                o1 = out1.cpu().numpy()
                h1, wn = o1[:mj], float(o1[mj])
                Gm = G[:mj, :mj]
                c = h1 + (h1 - Gm @ h1)
                s1, s2 = float(c @ h1), float(c @ (Gm @ c))
                eta2 = (wn - s1) - (s1 - s2)
                explicit = not (eta2 >= 1e-6 * wn) or not (wn > 0.0)
                cd = torch.from_numpy(np.ascontiguousarray(c)).to(dev)
                vnew = torch.empty_like(w)
                xnew = torch.empty_like(w)
                out2 = torch.empty(mj + 3, dtype=torch.float64, device=dev)
                yd = torch.zeros(mj, dtype=torch.float64, device=dev)
                if explicit:
                    # the norm formula cancelled: w - V c unscaled, its norm from the pass itself
                    _lib.call("bamg_cgs_update", _lib.ptr(table), mj, _lib.ptr(cd), _lib.ptr(yd), _lib.ptr(w),
                              _lib.ptr(x0), _lib.ptr(e), 1.0, 0, self.n_own, _lib.ptr(vnew), _lib.ptr(xnew),
                              _lib.ptr(out2))
                    part = out2[: mj + 2].clone()
                    self.comm.allreduce_(part)
                    eta2 = float(part[mj].item())
                h = np.empty(j + 2)
                h[:mj] = c
                h[mj] = np.sqrt(max(eta2, 0.0))
                happy = h[mj] <= 1e-14 * beta
                for i in range(j):
                    t = cs[i] * h[i] + sn[i] * h[i + 1]
                    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
                    h[i] = t
                rad = np.hypot(h[j], h[j + 1])
                cs[j], sn[j] = (1.0, 0.0) if rad == 0.0 else (h[j] / rad, h[j + 1] / rad)
                R[: j + 1, j] = h[: j + 1]
                R[j, j] = rad
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                its += 1
                used = mj
                y = solve_triangular(R[:used, :used], g[:used], lower=False)
                yd = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
                eta = float(np.sqrt(max(eta2, 0.0)))
                inv = 1.0 / eta if eta > 0.0 else 1.0
                if explicit:
                    # scale the unscaled w - V c kept above; x through the same pass with c = 0
                    if not happy:
                        vnew = _lincomb([vnew], [inv])
                    zero_c = torch.zeros(mj, dtype=torch.float64, device=dev)
                    scratch = torch.empty_like(w)
                    outx = torch.empty(mj + 3, dtype=torch.float64, device=dev)
                    _lib.call("bamg_cgs_update", _lib.ptr(table), mj, _lib.ptr(zero_c), _lib.ptr(yd), _lib.ptr(w),
                              _lib.ptr(x0), _lib.ptr(e), 1.0, 1, self.n_own, _lib.ptr(scratch), _lib.ptr(xnew),
                              _lib.ptr(outx))
                    out2[mj + 1] = outx[mj + 1]
                else:
                    _lib.call("bamg_cgs_update", _lib.ptr(table), mj, _lib.ptr(cd), _lib.ptr(yd), _lib.ptr(w),
                              _lib.ptr(x0), _lib.ptr(e), inv, int(happy), self.n_own, _lib.ptr(vnew),
                              _lib.ptr(xnew), _lib.ptr(out2))
                x = xnew
                out2[mj + 2 : mj + 3] = self._bx_norm2_local(x)
                self.comm.allreduce_(out2)
                o2 = out2.cpu().numpy()
                if not happy:
                    V.append(vnew)
                    G[:mj, mj] = G[mj, :mj] = o2[:mj] * inv
                    G[mj, mj] = o2[mj] * inv * inv
                nx = np.sqrt(o2[mj + 1])
                hist.append(np.inf if nx == 0.0 else float(np.sqrt(o2[mj + 2]) / nx))
                e_try = None  # formed on demand: e + V y
                if hist[-1] <= rtol:
                    done = True
                if done or happy or its >= max_iters:
                    done = done or happy
                    break
            # e <- e + V y (end of the cycle: converged, happy breakdown, restart or the cap)
            tab = self._table(V[:used])
            e_new = torch.empty_like(e)
            _lib.call("bamg_combine", _lib.ptr(tab), used, _lib.ptr(yd), None, _lib.ptr(e), self.n_own,
                      _lib.ptr(e_new))
            e = e_new
            x = _lincomb([e], [1.0], base=x0)
        return its, hist, done, x

    def gather(self, x_own):
        """Full l1-normalised, sign-fixed solution on every rank."""
        full = self.comm.all_gather_vec(x_own, self.part)
        return engine.sign_fix_l1(full)
