"""Worker functions for the multi-process tests (importable by spawned ranks)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def _init(rank, world, port, backend="gloo"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def plan_worker(rank, world, port, out_dir):
    """CPU: halo plans of every operator of a golden hierarchy + a host SpMV
    through the plans (gloo p2p) reproduces the global product bit for bit."""
    import torch
    from conftest import csr_from, load_golden
    from paper_1402_4005_b200.distributed import Comm, RowPartition, localize_host
    dist = _init(rank, world, port)
    comm = Comm()
    g = load_golden("pipe_uniform63")
    res = {}
    rng = np.random.default_rng(3)
    for key, rows_lv, cols_lv in (("L0_B", 0, 0), ("L0_Q", 1, 0), ("L0_P", 0, 1), ("L1_B", 1, 1)):
        A = csr_from(g, key)
        rp = RowPartition(A.shape[0], world)
        cp = RowPartition(A.shape[1], world)
        indptr, cols, vals, n_ext, plan = localize_host(A, rp, cp, rank, comm)
        x = rng.standard_normal(A.shape[1])  # same on every rank (same seed)
        c0, c1 = cp.range(rank)
        x_ext = np.empty(n_ext)
        x_ext[: c1 - c0] = x[c0:c1]
        ops, staged = [], {}
        for peer in sorted(set(plan.send_local) | set(plan.recv_counts)):
            if peer in plan.send_local:
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(x_ext[plan.send_local[peer]].copy()), peer))
            if peer in plan.recv_counts:
                staged[peer] = torch.empty(plan.recv_counts[peer], dtype=torch.float64)
                ops.append(dist.P2POp(dist.irecv, staged[peer], peer))
        for r in (dist.batch_isend_irecv(ops) if ops else []):
            r.wait()
        for peer, t in staged.items():
            o = plan.n_own + plan.recv_offset[peer]
            x_ext[o:o + t.numel()] = t.numpy()
        from scipy import sparse as sp
        loc = sp.csr_array((vals, cols, indptr), shape=(indptr.size - 1, n_ext))
        y_loc = loc @ x_ext
        r0, r1 = rp.range(rank)
        res[key] = bool(np.array_equal(y_loc, (A @ x)[r0:r1]))
    np.save(Path(out_dir) / f"plan_{rank}.npy", np.array([res[k] for k in sorted(res)]))
    dist.destroy_process_group()


def solve_worker(rank, world, port, out_dir, name, agg, backend="gloo"):
    """GPU: distributed V-cycle + GMRES -- gloo: ranks share one device (host-staged
    halos); nccl: one device per rank (device-buffer p2p and all-reduce)."""
    import torch
    from conftest import csr_from, gmres_args, load_golden
    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200.chains import ChainProblem
    from paper_1402_4005_b200.distributed import Comm, DistSolver
    from test_gpu_pipeline import _setup_cfg
    _init(rank, world, port, backend)
    torch.cuda.set_device(rank if backend == "nccl" else 0)
    g = load_golden(name)
    B = csr_from(g, "B")
    prob = ChainProblem(A=None, B=B, n=B.shape[0], family=str(g["family"]), params={},
                        geometry=g["geometry"] if "geometry" in g else None)
    cfg = _setup_cfg(g)
    setup = pb.run_setup(prob, cfg, draws=(g["init_right_draw"], g["init_left_draw"]))
    ds = DistSolver(setup.hierarchy, cfg.smoother, Comm(), agglomerate_rows=agg)
    r0, r1 = ds.r0, ds.r1
    vin = torch.from_numpy(np.ascontiguousarray(g["vcycle_in"][r0:r1])).cuda()
    vout = ds.comm.all_gather_vec(ds.vc.apply(vin), ds.part).cpu().numpy()
    restart, max_iters, rtol = gmres_args(g)
    x0 = setup.dx0[r0:r1].contiguous()
    its, hist, conv, x = ds.solve(x0, restart, max_iters, rtol)
    xf = ds.gather(x).cpu().numpy()
    np.savez(Path(out_dir) / f"solve_{rank}.npz", vout=vout, x=xf, its=its, conv=int(conv),
             levels_partitioned=len(ds.vc.levels))
    import torch.distributed as dist
    dist.destroy_process_group()


def setup_worker(rank, world, port, out_dir, name, backend="gloo"):
    """GPU: run_setup with the bootstrap relaxation split by triplet slot over the ranks
    (ranks share the device under gloo).  Every rank must end with the reference's hierarchy:
    patterns bit-exact, values and x0 within the single-GPU tolerances."""
    import torch
    from conftest import csr_from, load_golden
    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200 import bootstrap
    from paper_1402_4005_b200.distributed import Comm
    from test_gpu_pipeline import _close, _problem, _same_pattern, _setup_cfg
    _init(rank, world, port, backend)
    torch.cuda.set_device(rank if backend == "nccl" else 0)
    bootstrap.SLOT_PARTITION_MIN_ROWS = 64  # partition every level of the desk-size fixture
    from paper_1402_4005_b200 import interp
    interp.ROW_PARTITION_MIN_ROWS = 64      # ... its LS fits (row blocks) and Galerkin products too
    g = load_golden(name)
    cfg = _setup_cfg(g)
    injected = int(g["cfg_ints"][13]) >= 0
    draws = (g["init_right_draw"], g["init_left_draw"]) if injected else None
    setup = pb.run_setup(_problem(g), cfg, draws=draws, comm=Comm())
    levels = setup.hierarchy.levels
    ok = len(levels) == int(g["n_levels"])
    worst = 0.0
    for li, lev in enumerate(levels):
        for key in ("B", "M", "N") + (("P", "Q") if lev.dP is not None else ()):
            ref = csr_from(g, f"L{li}_{key}")
            got = getattr(lev, key)
            ok = ok and _same_pattern(got, ref) and _close(got.data, ref.data, 1e-9)
        if lev.dP is not None:
            ok = ok and bool(np.array_equal(lev.split.coarse, g[f"L{li}_coarse"]))
    x0_err = float(np.abs(setup.x0 - g["x0"]).sum())
    np.savez(Path(out_dir) / f"setup_{rank}.npz", ok=int(ok), x0_err=x0_err, x0=setup.x0,
             fits=interp.PARTITION_STATS["fits"], products=interp.PARTITION_STATS["products"])
    import torch.distributed as dist
    dist.destroy_process_group()


def cols_worker(rank, world, port, out_dir):
    """CPU: the slot partition's column all-gather (uneven widths) and the host side of the
    Gram-form Arnoldi coefficients against explicit CGS2 on a random basis."""
    import torch
    from paper_1402_4005_b200.distributed import Comm, slot_bounds
    _init(rank, world, port)
    comm = Comm()
    ok = True
    for k in (16, 12, 7):
        b = slot_bounds(k, world)
        ok = ok and b[0] == 0 and b[-1] == k and bool(np.all(np.diff(b) >= 0))
        full = torch.arange(50 * k, dtype=torch.float64).reshape(50, k)
        own = full[:, int(b[rank]): int(b[rank + 1])].contiguous()
        ok = ok and bool(torch.equal(comm.all_gather_cols(own, b), full))
    # row-block pieces of a CSR product (multi-GPU Galerkin products / LS fits): slices of the
    # rows, all-gathered, give back the matrix
    from scipy import sparse as sp
    from paper_1402_4005_b200.device import DeviceCSR
    from paper_1402_4005_b200.distributed import RowPartition, row_slice
    M = sp.random(37, 23, density=0.2, random_state=5, format="csr")
    M.sort_indices()
    D = DeviceCSR(torch.from_numpy(M.indptr.astype(np.int32)), torch.from_numpy(M.indices.astype(np.int32)),
                  torch.from_numpy(M.data.copy()), M.shape)
    part = RowPartition(37, world)
    own = row_slice(D, *part.range(rank))
    r0, r1 = part.range(rank)
    ok = ok and own.shape == (r1 - r0, 23) and int(own.rowptr[-1]) == own.nnz
    full = comm.all_gather_csr_rows(own, part)
    ok = ok and bool(torch.equal(full.rowptr, D.rowptr)) and bool(torch.equal(full.col, D.col)) \
        and bool(torch.equal(full.val, D.val))
    flat = comm.all_gather_flat(torch.arange(rank + 2, dtype=torch.int32))
    ok = ok and flat.tolist() == [v for r in range(world) for v in range(r + 2)]
    np.save(Path(out_dir) / f"cols_{rank}.npy", np.array([ok]))
    import torch.distributed as dist
    dist.destroy_process_group()
