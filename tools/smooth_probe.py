"""Where the k-wide smoothing time goes at full size (development tool).

python tools/smooth_probe.py [--config cfg4]

Times, with CUDA events and no L2 flush (as in the pipeline): a homogeneous
k-wide Jacobi sweep on B and on B^T (with / without the per-column peak),
back-to-back alternating sweeps, and a whole bamg_smooth_block call.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_1402_4005_b200 import engine
from paper_1402_4005_b200.device import DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--reps", type=int, default=6)
a = ap.parse_args()
prob = bench.build_problem(a.config)
k = bench.CONFIGS[a.config][2]
A = DeviceCSR.from_host(prob.B)
At = engine.transpose(A)
n, nnz = A.shape[0], A.nnz
d = engine.diag(A)
skip = engine.degenerate_rows(A, d)
skip_t = engine.degenerate_rows(At, d)
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.rand((n, k), dtype=torch.float64, device="cuda", generator=g)
U = torch.rand((n, k), dtype=torch.float64, device="cuda", generator=g)
peak = torch.zeros(2 * k, dtype=torch.float64, device="cuda")
sig = torch.zeros(k, dtype=torch.float64, device="cuda")


def timed(fn, reps=a.reps):
    ts = []
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


hom = 4.0 * (n + 1) + 12.0 * nnz + 16.0 * k * n + 9.0 * n


def alt():
    engine.jacobi(A, d, skip, V)
    engine.jacobi(At, d, skip_t, U)


rows = [
    ("jacobi B hom", lambda: engine.jacobi(A, d, skip, V), hom),
    ("jacobi Bt hom", lambda: engine.jacobi(At, d, skip_t, U), hom),
    ("jacobi B hom peak", lambda: engine.jacobi(A, d, skip, V, peak=peak), hom),
    ("jacobi B inhom(b=U)", lambda: engine.jacobi(A, d, skip, V, b=U, b_scale=sig), hom + 8.0 * k * n),
    ("alternating B, Bt", alt, 2 * hom),
    ("smooth_block hom 3 sweeps", lambda: engine.smooth_block(A, At, None, None, d, skip, skip_t, U, V, sig, 3, 0.7,
                                                            0, smooth=2, refresh=0), 6 * hom + 32.0 * k * n),
    ("smooth_block inhom 3 sweeps + refresh", lambda: engine.smooth_block(A, At, None, None, d, skip, skip_t, U, V,
                                                                         sig, 3, 0.7, 1, smooth=1, refresh=1), 0),
    ("col_norms", lambda: engine.col_norms(V), 8.0 * k * n),
    ("normalize_cols", lambda: engine.normalize_cols(V), 24.0 * k * n),
    ("refresh_sigmas", lambda: engine.refresh_sigmas(A, None, None, U, V, sig), 4.0 * (n + 1) + 12.0 * nnz + 16.0 * k * n),
]
for label, fn, by in rows:
    ms = timed(fn)
    print(f"{label:40s} {ms * 1e3:10.1f} us   {by / ms / 1e6:8.1f} GB/s (algorithmic)", flush=True)
