"""Per-launch HBM throughput of the CSR row kernels on level-0 operators (development tool).

python tools/csr_bench.py [--configs cfg1,cfg2] [--reps 20]

For each config's B (and B^T) times SpMV (k=1), Jacobi (k=1, the V-cycle
sweep), SpMM and Jacobi at the config's k, with the L2 flushed (256 MB write)
before every timed launch; prints algorithmic GB/s (SURVEY §8(d) byte model,
the same figure csrc/sparse.cu hands the profiler) and the fraction of the
measured HBM peak.  BAMG_ROWS_IMPL=rows selects the thread-gather kernel.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1402_4005_b200 import engine
from paper_1402_4005_b200.device import DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg1,cfg2")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ks", default="", help="comma list of k to run (default: 1 and the config's k)")
ap.add_argument("--flush", default="read", choices=["read", "write", "none"],
                help="L2 flush before each timed launch: read 256 MB (clean lines), write 256 MB, or none")
a = ap.parse_args()
peak = bench.peaks()[0]
flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")


def do_flush():
    if a.flush == "read":
        sink.copy_(flush.sum())
    elif a.flush == "write":
        flush.fill_(1.0)


def timed(fn):
    ts = []
    for _ in range(a.reps + 2):
        do_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


for name in a.configs.split(","):
    prob = bench.build_problem(name)
    k = bench.CONFIGS[name][2]
    A = DeviceCSR.from_host(prob.B)
    At = engine.transpose(A)
    engine.attach_stencil(A)   # lattice operators: stencil tiles (BAMG_NO_STENCIL=1 disables)
    engine.attach_stencil(At)
    n, nnz = A.shape[0], A.nnz
    d = engine.diag(A)
    skip = engine.degenerate_rows(A, d)
    g = torch.Generator(device="cuda").manual_seed(0)
    ks = [int(x) for x in a.ks.split(",")] if a.ks else [1, k]
    for kk in ks:
        X = torch.rand((n, kk) if kk > 1 else (n,), dtype=torch.float64, device="cuda", generator=g)
        Bv = torch.rand_like(X)
        base = 4.0 * (n + 1) + 12.0 * nnz + 8.0 * kk * n + 8.0 * kk * n
        rows = [
            (f"spmm B k={kk}", lambda: engine.spmm(A, X), base),
            (f"spmm Bt k={kk}", lambda: engine.spmm(At, X), base),
            (f"jacobi B k={kk}", lambda: engine.jacobi(A, d, skip, X, b=Bv), base + 8.0 * kk * n + 9.0 * n),
        ]
        if kk > 1:
            pk = torch.zeros(kk, dtype=torch.float64, device="cuda")
            rows += [
                (f"jacobi B k={kk} hom", lambda: engine.jacobi(A, d, skip, X), base + 9.0 * n),
                (f"jacobi B k={kk} hom+peak", lambda: engine.jacobi(A, d, skip, X, peak=pk), base + 9.0 * n),
            ]
        # speed of light at this size: a device copy moving the same bytes (read + write)
        half = int(base // 16)
        src = torch.ones(half, dtype=torch.float64, device="cuda")
        dst = torch.empty_like(src)
        rows.append((f"copy {2 * half * 8 / 1e6:.0f}MB", lambda: dst.copy_(src), 16.0 * half))
        for label, fn, by in rows:
            ms = timed(fn)
            gbs = by / ms / 1e6
            print(json.dumps({"config": name, "op": label, "n": n, "nnz": nnz, "us": round(ms * 1e3, 2),
                              "alg_MB": round(by / 1e6, 1), "GBps": round(gbs, 1),
                              "frac": round(gbs / peak, 3)}), flush=True)
