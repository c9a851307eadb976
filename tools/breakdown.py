"""Phase breakdown of setup + solve on one config (development tool, syncs per phase)."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1402_4005_b200 as pb
from paper_1402_4005_b200 import bootstrap as bs, chains
from paper_1402_4005_b200.device import DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
import bench
fam, side, k, stop, restart, _ = bench.CONFIGS[a.config]
t = time.time()
prob = bench.build_problem(a.config)
print("gen", time.time() - t, flush=True)
cfg = bench.setup_config(a.config)
g = np.random.default_rng(0)
draws = (g.random((k, prob.n)), g.random((k, prob.n)))
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(draws[0].T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(draws[1].T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda()
P = chains.ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
gcfg = pb.GmresConfig(restart=restart, rtol=1e-8)
from paper_1402_4005_b200 import _lib
import ctypes as C
for rep in range(a.reps):
    if rep == a.reps - 1:
        _lib.lib().bamg_trace_enable(_lib.ctx(), 1)
    bs.PHASES = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    tv = float("nan")
    if rep < a.reps - 1:  # V-cycle timing stays out of the traced step
        b = torch.randn(prob.n, dtype=torch.float64, device="cuda")
        vop.apply(b); torch.cuda.synchronize()
        tv = time.perf_counter()
        for _ in range(10): vop.apply(b)
        torch.cuda.synchronize(); tv = (time.perf_counter() - tv) / 10
    levels = [(l.n, l.nnz) for l in setup.hierarchy.levels]
    free_b, total_b = torch.cuda.mem_get_info()
    print(json.dumps({"rep": rep, "mem_used_gb": round((total_b - free_b) / 1e9, 2),
                      "torch_reserved_gb": round(torch.cuda.memory_reserved() / 1e9, 2), "setup": t1 - t0, "pinv": t2 - t1, "gmres": t3 - t2, "its": r.iterations,
                      "hist": r.residual_history[-1], "vcycle_ms": tv * 1e3, "levels": levels,
                      "phases": {k2: round(v, 4) for k2, v in bs.PHASES.items()}}), flush=True)
buf = C.create_string_buffer(1 << 20)
_lib.lib().bamg_trace_dump(_lib.ctx(), buf, 1 << 20)
rows = [l.split("\t") for l in buf.value.decode().splitlines()]
rows.sort(key=lambda r: -float(r[1]))
tot = sum(float(r[1]) for r in rows)
print(f"TRACE total kernel ms {tot:.2f} launches {sum(int(r[2]) for r in rows)}")
for r in rows[:a.top]:
    print(f"{float(r[1]):10.3f} ms {int(r[2]):7d}  {r[0]}")
