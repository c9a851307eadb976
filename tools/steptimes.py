"""Wall time of consecutive bench steps with host-stall diagnostics (development tool).

Logs engine calls slower than BAMG_SLOWCALL_MS and Python GC pauses > 5 ms.
"""
import argparse, gc, json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--prof", action="store_true", help="engine family profiler over the steps (alg bytes per family)")
a = ap.parse_args()

_gc_t = [0.0]


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t[0] = time.perf_counter()
    else:
        dt = (time.perf_counter() - _gc_t[0]) * 1e3
        if dt > 5:
            print(f"[gc] gen{info['generation']} {dt:.1f} ms collected={info['collected']}", flush=True)


gc.callbacks.append(_gc_cb)
import bench
import paper_1402_4005_b200 as pb
from paper_1402_4005_b200 import bootstrap as bs
from paper_1402_4005_b200.chains import ChainProblem
from paper_1402_4005_b200.device import DeviceCSR

fam, size, k, stop, restart, desc = bench.CONFIGS[a.config]
prob = bench.build_problem(a.config)
cfg = bench.setup_config(a.config)
gcfg = pb.GmresConfig(restart=restart, rtol=bench.RTOL)
rh, lh = bench.draws_for(k, prob.n)
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(rh.T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(lh.T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda()
P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
from paper_1402_4005_b200 import _lib
import ctypes as C
if a.prof:
    _lib.lib().bamg_prof_enable(_lib.ctx(), (1 << 0) | (1 << 1) | (1 << 3) | (1 << 6))
for i in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
    t1 = time.perf_counter()
    vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    t2 = time.perf_counter()
    rep = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(json.dumps({"step": i, "total_ms": round((t4 - t0) * 1e3, 2), "setup_ms": round((t1 - t0) * 1e3, 2),
                      "vop_ms": round((t2 - t1) * 1e3, 2), "gmres_ms": round((t3 - t2) * 1e3, 2),
                      "tail_ms": round((t4 - t3) * 1e3, 2)}), flush=True)
if a.prof:
    def rd(fid):
        ms, cnt, by = C.c_double(), C.c_int64(), C.c_double()
        _lib.lib().bamg_prof_read(_lib.ctx(), fid, C.byref(ms), C.byref(cnt), C.byref(by))
        return ms.value, cnt.value, by.value
    # the CSR family = engine families 0 (coarse levels) + 6 (operators >= 2^18 rows)
    for fname, fids in (("csr_stream_spmv_spmm_jacobi", (0, 6)), ("ls_fit", (1,)),
                        ("gmres_cgs2_basis_passes", (3,))):
        ms, cnt, by = (sum(v) for v in zip(*(rd(f) for f in fids)))
        print(json.dumps({"family": fname, "ms": ms, "launches": cnt, "alg_bytes": by}), flush=True)
