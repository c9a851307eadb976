"""Benchmark: BAMG setup + AMG-preconditioned GMRES to ||Bx||/||x|| < 1e-8 on B200.

Contract (see the task statement): `python bench.py --gpus N --steps K
--warmup W [--impl reference] [--config cfgX]` prints ONE JSON line on rank 0.

A step is one full pass of the hot path over the workload: run_setup
(bootstrap AMG: smoothing, LS transfer operators, Galerkin products, coarsest
triplets) + VCycleOperator (coarsest pseudo-inverse) + preconditioned GMRES
to rtol 1e-8.  The default workload is BASELINE.json configs[4], the largest
single-GPU configuration (BASELINE.json's metric names no config): the tandem
queue 4095 x 4095 = 16,769,025 states, k = 16, seed-0 uniform(0,1) test
vectors, unrestarted GMRES.  The metric is a time: `value` = device seconds
per step with the operator, geometry and initial vectors resident in HBM
(`setup_s` / `solve_s` split it); `e2e` = the same through
`solve_steady_state` with host inputs (pinned H2D of B / draws / geometry and
the D2H of x inside the timed region).  `parity` compares the last step's
hierarchy and stationary vector with the reference-generated full-size
fixture (tests/golden/big_cfgX.npz) after the timed regions.

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N local ranks (127.0.0.1); under torchrun
WORLD_SIZE must equal N.  Each rank runs an independent replica of the
workload (`scaling: weak`; the setup is not partitioned yet, see DESIGN.md
section 6); `--partitioned` instead row-partitions the solve phase over NCCL
(paper_1402_4005_b200/distributed.py).  Every rank times its own steps with
CUDA events and rank 0 reports the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (family, side / n, k, stop_size override, gmres restart, description)
    "cfg0": ("tandem", 64, 8, 65, None, "tandem queue 64x64 (4,096 states), k=8, coarsest<=64"),
    "cfg1": ("uniform2d", 1023, 8, None, None, "uniform 2-D walk 1023x1023 (1,046,529 states), k=8"),
    "cfg2": ("tandem", 1024, 16, None, 30, "tandem queue 1024x1024 (1,048,576 states), k=16, GMRES(30)"),
    "cfg3": ("planar", 2 ** 21, 12, None, None, "random planar Delaunay chain, 2^21 states, k=12"),
    "cfg4": ("tandem", 4095, 16, None, None, "tandem queue 4095x4095 (16,769,025 states), k=16"),
}
DEFAULT_CONFIG = "cfg4"  # the largest single-GPU configuration of BASELINE.json
RTOL = 1e-8
METRIC = "AMG-GMRES setup+solve time to ||Bx||/||x||<1e-8 (s); V-cycle HBM GB/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def build_problem(name, validate=False):
    from paper_1402_4005_b200 import chains
    fam, size, k, stop, restart, _ = CONFIGS[name]
    if fam == "tandem":
        prob = chains.tandem_queue(size, validate=validate)
    elif fam == "uniform2d":
        prob = chains.uniform_2d(size, validate=validate)
    else:
        prob = chains.random_planar(size, seed=1, validate=validate)
    return prob


def setup_config(name):
    from dataclasses import replace

    from paper_1402_4005_b200 import default_setup_config
    fam, size, k, stop, restart, _ = CONFIGS[name]
    cfg = default_setup_config(fam, seed=0, n_tests=k)
    if stop is not None:
        cfg = replace(cfg, coarsening=replace(cfg.coarsening, stop_size=stop))
    return cfg


def draws_for(k, n):
    g = np.random.default_rng(0)  # BASELINE: k uniform(0,1) vectors, seed 0 (right, then left)
    return g.random((k, n)), g.random((k, n))


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    Polls NVML in-process (pynvml; ctypes calls release the GIL) every 50 ms
    -- forking nvidia-smi from a CUDA process stalls the host thread that
    issues the step's launches.  Falls back to nvidia-smi when pynvml is
    missing."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    BITS = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(index)
            try:
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv, h = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            return [str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in self.BITS]
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        return [v.strip() for v in out.split(",")] if out else None

    def _run(self):
        while not self._stop.is_set():
            try:
                row = self._sample()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            self._stop.wait(0.05 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() in ("active", "1")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def vcycle_bytes(levels, nu1, nu2, as_stored=False):
    """Algorithmic HBM bytes of one V-cycle (SURVEY.md section 8(d) model: 12 bytes per CSR
    entry).  `as_stored` counts a level whose operator carries the packed copy
    (bamg_csr_pack: 4 bytes per entry, no d / 1/d streams) at what its kernels really stream."""
    total = 0.0
    for li, lv in enumerate(levels[:-1]):
        n, nnz = lv.n, lv.nnz
        if as_stored and lv.dB.packed is not None:
            words = int(lv.dB.packed.numel())  # slice-major words incl. padding; offsets per 32 rows
            opb = 4 * words + 4 * (n // 32 + 1)
            if lv.dB.ptiles is not None:
                # stencil tiles read a flag per 256 rows instead of their words and offsets
                opb = opb * (1.0 - 256.0 * int(lv.dB.stencil.st_tiles) / n) + n / 256
            sweep = opb + 25 * n
            resid = opb + 24 * n
        else:
            sweep = 12 * nnz + 4 * (n + 1) + 32 * n
            resid = 12 * nnz + 4 * (n + 1) + 24 * n
        first = 24 * n
        nc = levels[li + 1].n
        restrict = 12 * lv.dQ.nnz + 4 * (nc + 1) + 8 * n + 8 * nc
        prolong = 12 * lv.dP.nnz + 4 * (n + 1) + 8 * nc + 16 * n
        total += first + (nu1 - 1 + nu2) * sweep + resid + restrict + prolong
    nl = levels[-1].n
    total += 8 * (nl + 1) ** 2 + 16 * (nl + 1)
    return total


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200 import _lib
    from paper_1402_4005_b200.chains import ChainProblem
    from paper_1402_4005_b200.device import DeviceCSR

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    name = args.config
    fam, size, k, stop, restart, desc = CONFIGS[name]
    prob = build_problem(name)
    n = prob.n
    cfg = setup_config(name)
    gcfg = pb.GmresConfig(restart=restart, rtol=RTOL)
    right_h, left_h = draws_for(k, n)

    # ---- inputs resident in HBM for the device-timed `value`
    dB = DeviceCSR.from_host(prob.B)
    dV = torch.from_numpy(np.ascontiguousarray(right_h.T)).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(left_h.T)).cuda()
    dgeo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda() if prob.geometry is not None else None
    dprob = ChainProblem(A=None, B=dB, n=n, family=fam, params={}, geometry=dgeo)
    zero = torch.zeros(n, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    c = _lib.ctx()
    partitioned = world > 1 and args.partitioned
    stream = torch.cuda.current_stream()

    class _Rep:
        def __init__(self, its, hist, conv):
            self.iterations, self.residual_history, self.converged = its, hist, conv

    setup_comm = None
    if partitioned:
        from paper_1402_4005_b200.distributed import Comm
        setup_comm = Comm()

    def step(mark=None):
        # partitioned: the bootstrap relaxation is split by triplet slot over the ranks
        setup = pb.run_setup(dprob, cfg, draws=(dV, dU), B_device=dB, comm=setup_comm)
        if mark is not None:
            mark.record(stream)
        if partitioned:
            # row-partitioned V-cycle + GMRES over NCCL (setup replicated per rank)
            from paper_1402_4005_b200.distributed import Comm, DistSolver
            ds = DistSolver(setup.hierarchy, cfg.smoother, Comm())
            its, hist, conv, x = ds.solve(setup.dx0[ds.r0:ds.r1].contiguous(), restart, 1000, RTOL)
            return setup, ds, _Rep(its, hist, conv)
        vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
        rep = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
        return setup, vop, rep

    for _ in range(args.warmup):
        setup, vop, rep = step()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- device-timed region: K steps, barrier + sync both sides
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = int(L.bamg_launch_count(c))
    import gc
    gc.collect()  # host housekeeping before the timed region, not inside it
    gc.disable()
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        iters = []
        marks, mids = [], []
        for _ in range(args.steps):
            mids.append(torch.cuda.Event(enable_timing=True))
            setup, vop, rep = step(mark=mids[-1])
            iters.append(rep.iterations)
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    gc.enable()
    launches = int(L.bamg_launch_count(c)) - launches0
    dev_s = ev0.elapsed_time(ev1) / 1e3 / args.steps
    starts = [ev0] + marks[:-1]
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, marks)]
    setup_ms = [a.elapsed_time(b) for a, b in zip(starts, mids)]
    solve_ms = [a.elapsed_time(b) for a, b in zip(mids, marks)]
    if dist is not None:
        t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    converged = bool(rep.converged) and rep.residual_history[-1] < RTOL

    # ---- roofline window: the same K steps again with the engine profiler on
    # (CUDA events around every launch of the CSR row family, the LS fit and
    # the GMRES orthogonalisation passes on the engine's stream).  The events
    # cost time, so `value` comes from the un-instrumented region above and the
    # per-launch kernel times from this one.
    FAMS = {0: "csr", 1: "ls_fit", 3: "gmres_ortho", 6: "csr_fine"}
    L.bamg_prof_enable(c, sum(1 << f for f in FAMS))
    gc.collect()
    gc.disable()
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    barrier()
    gc.enable()
    import ctypes as C
    raw = {}
    for fid in FAMS:
        ms, cnt, by = C.c_double(), C.c_int64(), C.c_double()
        L.bamg_prof_read(c, fid, C.byref(ms), C.byref(cnt), C.byref(by))
        raw[fid] = (ms.value, cnt.value, by.value)
    L.bamg_prof_enable(c, 0)
    fam_stats = {
        # the CSR family = its launches on every level (engine families 0 + 6)
        "csr_stream_spmv_spmm_jacobi": tuple(a + b for a, b in zip(raw[0], raw[6])),
        "gmres_cgs2_basis_passes": raw[3],
        "ls_fit": raw[1],
    }
    fine = raw[6]

    # ---- V-cycle throughput (secondary metric of BASELINE.json)
    levels = setup.hierarchy.levels
    if partitioned:
        vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    vb_csr = vcycle_bytes(levels, cfg.smoother.sweeps_pre, cfg.smoother.sweeps_post)
    vb = vcycle_bytes(levels, cfg.smoother.sweeps_pre, cfg.smoother.sweeps_post, as_stored=True)
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        vop.apply(b)
    nv = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(nv):
        vop.apply(b)
    e1.record(stream)
    torch.cuda.synchronize()
    vms = e0.elapsed_time(e1) / nv
    peak, peak_kind = peaks()

    # ---- parity of the last timed step against the reference's full-size fixture
    parity = None
    if not args.no_parity and rank == 0:
        try:
            sys.path.insert(0, str(ROOT / "tests"))
            import bigparity
            res = bigparity.check_config(name, result=(prob, dB, cfg, setup))
            parity = {k_: res.get(k_) for k_ in ("ok", "why", "mode", "operators_checked", "iterations",
                                                  "reference_iterations", "gmres_start", "x_err_l1",
                                                  "x_err_l1_est", "x_err_l1_blocks", "vcycle_err_rel",
                                                  "failures") if k_ in res}
            parity["fixture"] = f"tests/golden/big_{name}.npz (unmodified reference, tests/golden/make_golden_big.py)"
            del res
        except Exception as exc:  # parity is reported, never fatal to the timing line
            parity = {"ok": None, "why": f"{type(exc).__name__}: {exc}"}
        torch.cuda.empty_cache()

    # ---- e2e through the public API with host inputs
    # the user's inputs are the chain (B, geometry) and the config: the seeded
    # uniform(0,1) test vectors are drawn inside the call on the device
    # (run_setup(draws="uniform"), numpy's PCG64 bit for bit), as the reference
    # draws its test vectors inside run_setup from cfg.seed
    Bh = prob.B
    pins = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in
            (Bh.indptr.astype(np.int32), Bh.indices.astype(np.int32), Bh.data,
             np.ascontiguousarray(prob.geometry.T))]
    h2d = sum(t.numel() * t.element_size() for t in pins)
    xout = torch.empty(n, dtype=torch.float64).pin_memory()
    d2h = xout.numel() * 8

    copy_stream = torch.cuda.Stream()

    def e2e_step():
        # every input goes over a copy stream: B first (ChainProblem.B_ready: the setup draws its
        # seeded test vectors while it lands), then the coordinates, which are first read at the
        # first C/F split, after the initial relaxation (ChainProblem.geometry_ready)
        b_ready, g_ready = torch.cuda.Event(), torch.cuda.Event()
        copy_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(copy_stream):
            rp, ci, va = [t.to("cuda", non_blocking=True) for t in pins[:3]]
            b_ready.record(copy_stream)
            ge = pins[3].to("cuda", non_blocking=True)
            g_ready.record(copy_stream)
        for t in (rp, ci, va, ge):
            t.record_stream(torch.cuda.current_stream())
        B = DeviceCSR(rp, ci, va, Bh.shape)
        p = ChainProblem(A=None, B=B, n=n, family=fam, params={}, geometry=ge, geometry_ready=g_ready,
                         B_ready=b_ready)
        rep2 = pb.solve_steady_state(p, cfg, gcfg, draws="uniform", to_host=False)
        xout.copy_(rep2.x_device, non_blocking=True)
        torch.cuda.synchronize()
        return rep2

    for _ in range(max(1, args.warmup)):  # untimed: the caching allocator settles on the e2e path's buffers
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        rep2 = e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_s = max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- dominant kernel family -> roofline
    def fam_json(v):
        ms, cnt, by = v
        if not cnt:
            return {"ms_per_step": 0.0, "launches_per_step": 0}
        per = ms / 1e3 / cnt
        return {"ms_per_step": round(ms / args.steps, 3), "launches_per_step": cnt // args.steps,
                "alg_bytes_per_launch": round(by / cnt), "alg_GBps": round((by / cnt) / per / 1e9, 1) if per else 0.0,
                "frac_of_hbm_peak": round((by / cnt) / per / 1e9 / peak, 4) if per else 0.0}

    hbm_fams = {k_: v for k_, v in fam_stats.items() if k_ != "ls_fit"}
    dom = max(hbm_fams, key=lambda f: hbm_fams[f][0])
    ms, cnt, by = fam_stats[dom]
    per_launch_s = ms / 1e3 / max(cnt, 1)
    achieved = (by / max(cnt, 1)) / per_launch_s / 1e9 if cnt else 0.0
    traffic, traffic_src = family_traffic(dom, by / max(cnt, 1))
    roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
            "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
            "alg_bytes_per_launch": round(by / max(cnt, 1)),
            "launches_in_window": cnt, "share_of_step": round(ms / 1e3 / (dev_s * args.steps), 4),
            "window": f"{args.steps} profiled steps after the timed region (same workload)",
            "families": {f: fam_json(v) for f, v in fam_stats.items()}}
    fit = fp64_fit_roofline(L, c, fam_stats.get("ls_fit"), args.steps, name)
    if fit:
        roof["ls_fit_fp64"] = fit
    if fine[1]:
        # the CSR family restricted to the finest levels (operators >= 2^18 rows):
        # bandwidth-sized launches, without the latency-bound coarse-level ones
        fa = (fine[2] / fine[1]) / (fine[0] / 1e3 / fine[1]) / 1e9
        roof["finest_levels"] = {"rows_min": 1 << 18, "launches": fine[1], "ms_total": round(fine[0], 3),
                                 "alg_bytes_per_launch": round(fine[2] / fine[1]), "achieved": round(fa, 1),
                                 "frac": round(fa / peak, 4)}
    line = {
        "metric": METRIC, "value": round(dev_s, 6), "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_s * 1e3, 3),
        "higher_is_better": False, "scaling": "strong" if partitioned else "weak", "vs_baseline": None,
        "dtype": "f64",
        "setup_s": round(float(np.mean(setup_ms)) / 1e3, 6), "solve_s": round(float(np.mean(solve_ms)) / 1e3, 6),
        "step_ms": {"min": round(min(step_ms), 3), "median": round(float(np.median(step_ms)), 3),
                    "max": round(max(step_ms), 3)},
        "data": "synthetic: BASELINE generator chain, seed-0 uniform(0,1) test vectors",
        "config": {"workload": f"{name}: {desc}", "n": n, "nnz": int(dB.nnz), "k": k,
                   "gmres_restart": restart, "rtol": RTOL, "setup_cycles": cfg.setup_cycles,
                   "levels": [lv.n for lv in levels], "gmres_iterations": iters[-1],
                   "converged": converged,
                   "parallelism": (f"row-partitioned V-cycle+GMRES over NCCL x{world}; setup: bootstrap relaxation "
                                   "slot-partitioned, fits / Galerkin products / coarsest replicated"
                                   if partitioned else f"independent replicas x{world}"),
                   "l2": "working set (operators + k-vector blocks) > 126 MB L2; no flush"},
        # bytes as stored (level 0 streams its packed 4-byte entries); csr_model_bytes is SURVEY 8(d)'s
        # 12-bytes-per-entry figure for the same V-cycle, for comparison with earlier rounds
        "vcycle": {"ms": round(vms, 4), "alg_bytes": int(vb), "GBps": round(vb / (vms / 1e3) / 1e9, 1),
                   "frac_of_hbm_peak": round(vb / (vms / 1e3) / 1e9 / peak, 4),
                   "csr_model_bytes": int(vb_csr),
                   "csr_model_GBps": round(vb_csr / (vms / 1e3) / 1e9, 1)},
        "roofline": roof,
        "e2e": {"value": round(e2e_s, 6), "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "parity": parity,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, args.cpu_sample)
    if dist is not None:
        dist.destroy_process_group()
    return line


def fp64_fit_roofline(L, c, fam, steps, name):
    """The LS fit against the fp64 CUDA-core peak.

    flops per step: ncu's thread-level DFMA/DADD/DMUL counts over every fit
    launch of one cfg1 step (profiles/rNN_ls_fit_flops.json, tools/fit_flops.py;
    the fit is deterministic, so the count is the same every step).  time: the
    fit family's live CUDA-event total over the profiled window.  peak: the DFMA
    throughput probe (bamg_fp64_peak) run here, on this GPU."""
    files = sorted(ROOT.glob("profiles/r*_ls_fit_flops.json"))
    if not fam or not fam[1] or name != "cfg1" or not files:
        return None
    import ctypes as C
    pk = C.c_double()
    if L.bamg_fp64_peak(c, 5, C.byref(pk)) != 0:
        return None
    d = json.load(open(files[-1]))
    fl = d["fp64_flops_per_step"]
    ach = fl * steps / (fam[0] / 1e3) / 1e12
    return {"bound": "fp64 latency", "achieved": round(ach, 3), "peak": round(pk.value, 2), "unit": "TFLOP/s",
            "frac": round(ach / pk.value, 4), "flops_per_step": fl, "ms_per_step": round(fam[0] / steps, 3),
            "alg_GBps": round(fam[2] / (fam[0] / 1e3) / 1e9, 1),
            "peak_kind": "measured live (bamg_fp64_peak: DFMA chains, full occupancy)",
            "flops_source": f"{files[-1].name}: ncu thread-level fp64 instruction counts, one step"}


def family_traffic(family, alg_per_launch):
    """roofline.traffic: DRAM bytes per launch of the roofline's kernel family.

    From the committed ncu capture (profiles/rNN_family_traffic.json, made by
    tools/family_traffic.py): ncu's dram__bytes_read.sum + dram__bytes_write.sum
    over every launch of the family in one graph-free step, divided by the
    engine's algorithmic bytes for the same launches.  The timed region's
    launches get that measured traffic/algorithmic ratio applied to their own
    algorithmic bytes per launch."""
    for f in sorted(ROOT.glob("profiles/r*_family_traffic.json"), reverse=True):
        d = json.load(open(f))
        e = d.get("families", {}).get(family)
        if e and e.get("traffic_over_alg"):
            ratio = e["traffic_over_alg"]
            return round(alg_per_launch * ratio), (f"{f.name}: ncu DRAM bytes / algorithmic bytes = {ratio:.3f} "
                                                   f"over {e['launches']} launches of one {d.get('config')} step, "
                                                   f"applied per launch")
    return None, None


SAMPLES = {"tandem": 128, "uniform2d": 127, "planar": 4096}  # side (lattices) or n (planar)


def reference_calibration():
    """profiles/r*_reference_calibration.json: per config, the full-size run of
    the UNMODIFIED reference (tests/golden/make_golden_big.py, this build
    container, single-core-equivalent seconds) over the linear extrapolation
    of the port's bounded sample timed on the same machine (tools/ref_calibration.py)."""
    files = sorted(ROOT.glob("profiles/r*_reference_calibration.json"))
    if not files:
        return {}, None
    return json.loads(files[-1].read_text()).get("configs", {}), files[-1].name


def cpu_baseline(name, sample=None, repeat=1):
    """The oracle (numpy restatement of the reference, bit-identical to it on the
    golden fixtures) timed on a bounded sample of the same family on ONE host
    core (the reference is single-threaded: SURVEY.md section 8(b)), then
    extrapolated to the full workload: linear in the state count, times the
    calibration factor measured against a full-size run of the unmodified
    reference (`calibration`).  `value_kind` says so; the sample's own time is
    `sample_seconds`."""
    sys.path.insert(0, str(ROOT))
    from threadpoolctl import threadpool_limits

    from oracle import bamg_oracle as orc
    fam, size, k, stop, restart, desc = CONFIGS[name]
    from paper_1402_4005_b200 import chains
    if fam == "planar":
        n_s = sample or SAMPLES[fam]
        prob = chains.random_planar(n_s, seed=1, validate=False)
        n_full = size
    else:
        side = sample or SAMPLES[fam]
        prob = chains.tandem_queue(side, validate=False) if fam == "tandem" else chains.uniform_2d(side, validate=False)
        n_s = prob.n
        n_full = size * size
    cfg = orc.default_cfg(fam, k=k, stop=stop, seed=0)
    right, left = draws_for(k, prob.n)
    best = None
    with threadpool_limits(1):
        for _ in range(repeat):
            t0 = time.perf_counter()
            levels, T, x0, its, hist, conv, x = orc.solve(prob.B, cfg, prob.geometry, right, left, restart, RTOL)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
    cal, src = reference_calibration()
    entry = cal.get(name)
    factor = float(entry["factor"]) if entry else 1.0
    out = {"value": round(best * n_full / n_s * factor, 2), "unit": "s", "cores": 1, "kind": "port",
           "value_kind": "extrapolated: sample seconds x (n_full / n_sample) x calibration factor",
           "sample_seconds": round(best, 3),
           "sample": f"oracle (numpy/scipy restatement, 1 thread) setup+solve on {fam} n={n_s} "
                     f"({best:.2f} s, {its} GMRES its), scaled x{n_full / n_s:.1f} linearly in n to n={n_full}"}
    if entry:
        out["calibration"] = dict(entry, source=src)
    else:
        out["calibration"] = {"factor": 1.0, "note": "no full-size reference run for this config"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port; /root/reference is not on the GPU box) on one host core, rank
    0 only; each step a bounded sample of the workload, extrapolated as
    cpu_baseline() says."""
    if rank != 0:
        return None
    name = args.config
    for _ in range(args.warmup):
        cpu_baseline(name, args.cpu_sample)
    vals, samples = [], []
    for _ in range(args.steps):
        cb = cpu_baseline(name, args.cpu_sample)
        vals.append(cb["value"])
        samples.append(cb["sample_seconds"])
    v = float(np.mean(vals))
    fam, size, k, stop, restart, desc = CONFIGS[name]
    cb = dict(cb, value=round(v, 2), sample_seconds=round(float(np.mean(samples)), 3))
    return {"metric": METRIC, "value": round(v, 2), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "value_kind": cb["value_kind"],
            "data": "synthetic: BASELINE generator chain, seed-0 uniform(0,1) test vectors",
            "config": {"workload": f"{name}: {desc}", "k": k, "gmres_restart": restart, "rtol": RTOL},
            "cpu_baseline": cb,
            "e2e": {"value": round(v, 2), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def relaunch_under_torchrun(args_list, n):
    """`--gpus N` outside torchrun: run this script under torch.distributed.run
    with N local ranks (127.0.0.1) and pass its exit code through."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + args_list
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="N>1: row-partition the solve over NCCL instead of independent replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(sys.argv[1:], args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
