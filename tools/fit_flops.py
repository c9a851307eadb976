"""fp64 work of the LS fit (development tool, run under ncu).

python tools/fit_flops.py [--config cfg1] [--steps 1]

Runs bench.py's step (setup + V-cycle operator + GMRES) `steps` times and
prints the fp64 FMA peak the engine measures (`bamg_fp64_peak`).  Under

  ncu --kernel-name regex:fit_rows --metrics \
      sm__sass_thread_inst_executed_op_dfma_pred_on.sum,\
      sm__sass_thread_inst_executed_op_dadd_pred_on.sum,\
      sm__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum \
      --csv --log-file fit.csv python tools/fit_flops.py --steps 1

the launch list gives the LS fit's fp64 flops per step (2 per DFMA, 1 per
DADD/DMUL), which bench.py divides by the live fit time
(profiles/r01_ls_fit_flops.json).
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
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()

fam, size, k, stop, restart, _ = bench.CONFIGS[a.config]
prob = bench.build_problem(a.config)
cfg = bench.setup_config(a.config)
gcfg = pb.GmresConfig(restart=restart, rtol=bench.RTOL)
right, left = bench.draws_for(k, prob.n)
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(right.T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(left.T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda() if prob.geometry is not None else None
P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
for _ in range(a.steps):
    setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
    vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    r = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
torch.cuda.synchronize()
t = C.c_double()
L, c = _lib.lib(), _lib.ctx()
assert L.bamg_fp64_peak(c, 5, C.byref(t)) == 0, _lib.last_error() if hasattr(_lib, "last_error") else ""
print(f"fp64_peak_tflops {t.value:.2f}")
