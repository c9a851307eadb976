"""Run BASELINE configs end to end on the GPU: timings (best of 3 repetitions, host-
synchronised), iterations, invariants.

python tools/run_configs.py cfg0 cfg1 cfg2 cfg3 cfg4
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_1402_4005_b200 as pb
from paper_1402_4005_b200 import engine
from paper_1402_4005_b200.chains import ChainProblem
from paper_1402_4005_b200.device import DeviceCSR


def invariants(setup):
    """1^T B_l = 0 (column sums), 1^T Q = 1^T, P = I on C points (test_acceptance.py:150-176)."""
    worst_col, worst_q, p_ident = 0.0, 0.0, True
    for lv in setup.hierarchy.levels:
        B = lv.dB
        ones = torch.ones(B.shape[0], dtype=torch.float64, device="cuda")
        Bt = engine.transpose(B)
        cs = engine.spmm(Bt, ones)
        worst_col = max(worst_col, float(cs.abs().max()) / max(float(B.val.abs().max()), 1e-300))
        if lv.dQ is not None:
            W = lv.dW
            qs = engine.spmm(engine.transpose(lv.dQ), torch.ones(lv.dQ.shape[0], dtype=torch.float64, device="cuda"))
            worst_q = max(worst_q, float((qs - 1.0).abs().max()))
    return worst_col, worst_q


def main(names):
    for name in names:
        t = time.time()
        prob = bench.build_problem(name)
        gen = time.time() - t
        cfg = bench.setup_config(name)
        fam, size, k, stop, restart, desc = bench.CONFIGS[name]
        right, left = bench.draws_for(k, prob.n)
        dB = DeviceCSR.from_host(prob.B)
        dV = torch.from_numpy(np.ascontiguousarray(right.T)).cuda()
        dU = torch.from_numpy(np.ascontiguousarray(left.T)).cuda()
        geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda()
        P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
        gcfg = pb.GmresConfig(restart=restart, rtol=1e-8)
        out = {}
        import gc
        best = None
        for rep in range(3):
            gc.collect()  # no collector pause inside the timed repetition (as bench.py)
            gc.disable()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
            zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
            rep_ = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            if best is not None and (t2 - t0) >= best:
                gc.enable()
                continue
            best = t2 - t0
            out = {"config": name, "n": prob.n, "gen_s": round(gen, 2), "setup_s": round(t1 - t0, 4),
                   "solve_s": round(t2 - t1, 4), "its": rep_.iterations, "converged": rep_.converged,
                   "final": rep_.residual_history[-1], "levels": [lv.n for lv in setup.hierarchy.levels],
                   "o_c": round(pb.complexities(setup.hierarchy)[1], 3)}
            gc.enable()
        x = engine.sign_fix_l1(rep_.x_device)
        out["x_min"] = float(x.min())
        wc, wq = invariants(setup)
        out["worst_colsum_rel"] = wc
        out["worst_1TQ_dev"] = wq
        out["mem_GB"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
        print(json.dumps(out), flush=True)
        del setup, vop, rep_, P, dB, dV, dU
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg0", "cfg1", "cfg2"])
