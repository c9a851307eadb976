"""cProfile of the steady-state bench step (host-side cost; development aid)."""
import cProfile, io, pstats, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
import paper_1402_4005_b200 as pb
from paper_1402_4005_b200.chains import ChainProblem
from paper_1402_4005_b200.device import DeviceCSR

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
fam, size, k, stop, restart, desc = bench.CONFIGS[name]
prob = bench.build_problem(name)
cfg = bench.setup_config(name)
gcfg = pb.GmresConfig(restart=restart, rtol=bench.RTOL)
rh, lh = bench.draws_for(k, prob.n)
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(rh.T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(lh.T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda()
P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")


def step():
    setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
    vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    return pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)


for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(35)
print(s.getvalue())
