"""Time the coarsest dense pipeline (pinv + coarsest triplets) at n in {256, 1024}."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1402_4005_b200 import engine, chains
from paper_1402_4005_b200.device import DeviceCSR
sides = [int(a) for a in sys.argv[1:]] or [16, 32]
for side in sides:
    prob = chains.tandem_queue(side, validate=False)
    B = DeviceCSR.from_host(prob.B)
    D = engine.csr_to_dense(B)
    I = DeviceCSR.identity(prob.n)
    M = engine.csr_to_dense(I)
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        Z = engine.dense_pinv(D, prob.n)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        U, V, s, _ = engine.coarsest_triplets(D, M, M, prob.n, 16)
        torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"n={prob.n} pinv {1e3*(t1-t):.2f} ms triplets {1e3*(t2-t1):.2f} ms sig0={s[0].item():.3e} sig1={s[1].item():.3e}", flush=True)
