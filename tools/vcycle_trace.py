"""Per-launch device times of one V-cycle (development tool).

python tools/vcycle_trace.py [--config cfg1]

Builds the hierarchy once, then runs one V-cycle with the engine trace on
(graphs off: every launch bracketed by CUDA events; ~1-2 us of event overhead
each) and prints the launches in order with their duration, plus the sums per
level (launch order follows the level walk: down 0..L-2, coarsest, up L-2..0).
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
import paper_1402_4005_b200 as pb
from paper_1402_4005_b200 import _lib
from paper_1402_4005_b200.chains import ChainProblem
from paper_1402_4005_b200.device import DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
a = ap.parse_args()
fam, size, k, stop, restart, _ = bench.CONFIGS[a.config]
prob = bench.build_problem(a.config)
cfg = bench.setup_config(a.config)
right, left = bench.draws_for(k, prob.n)
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(right.T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(left.T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda() if prob.geometry is not None else None
P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
b = torch.randn(prob.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    vop.apply(b)
torch.cuda.synchronize()
L, c = _lib.lib(), _lib.ctx()
L.bamg_trace_enable(c, 1)
vop.apply(b)
torch.cuda.synchronize()
buf = C.create_string_buffer(1 << 20)
L.bamg_trace_timeline(c, buf, 1 << 20)
L.bamg_trace_enable(c, 0)
rows = [r.split("\t") for r in buf.value.decode().splitlines()]
ev = [(r[0], float(r[1]), float(r[2])) for r in rows]
levels = [lv.n for lv in setup.hierarchy.levels]
print("levels:", levels)
t0 = ev[0][1]
for name, s, e in ev:
    print(f"{(s - t0):9.1f} {e - s:7.1f} us  {name[:70]}")
print(f"span {(ev[-1][2] - t0):.1f} us, kernel-busy {sum(e - s for _, s, e in ev):.1f} us, {len(ev)} launches")
