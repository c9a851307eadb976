import sys, os
sys.path.insert(0, ".")
os.environ["BAMG_DEBUG"] = "1"
import numpy as np, torch
import bench
import paper_1402_4005_b200 as pb
from paper_1402_4005_b200 import bootstrap as bs
# stop before the dense solve: monkeypatch coarsest_triplets to report and abort
class Stop(Exception): pass
def fake(B, M, N, r):
    print(f"[probe] coarsest n={pb.sparse.as_device(B).shape[0]}", flush=True)
    raise Stop()
bs.coarsest_triplets = fake
name = sys.argv[1]
prob = bench.build_problem(name)
cfg = bench.setup_config(name)
fam, size, k, stop, restart, desc = bench.CONFIGS[name]
right, left = bench.draws_for(k, prob.n)
try:
    pb.run_setup(prob, cfg, draws=(right, left))
except Stop:
    pass
