"""Packed (bamg_csr_pack) vs plain CSR k = 1 kernels on a config's level-0 B (development tool)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_1402_4005_b200 import _lib, engine
from paper_1402_4005_b200.device import DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
prob = bench.build_problem(a.config)
plain = DeviceCSR.from_host(prob.B)
packed = DeviceCSR(plain.rowptr, plain.col, plain.val, plain.shape)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); ok = engine.pack_operator(packed); t1.record(); torch.cuda.synchronize()
print("packed:", ok, f"{t0.elapsed_time(t1):.3f} ms (first call)")
t0.record(); ok = engine.pack_operator(packed); t1.record(); torch.cuda.synchronize()
print("packed:", ok, f"{t0.elapsed_time(t1):.3f} ms")
n, nnz = plain.shape[0], plain.nnz
d = engine.diag(plain)
skip = engine.degenerate_rows(plain, d)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
r = torch.empty_like(x)


def timed(fn):
    ts = []
    for _ in range(a.reps + 2):
        sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


for name, A, mb in (("plain", plain, 12.0), ("packed", packed, 4.0)):
    base = 4.0 * (n + 1) + mb * nnz + 16.0 * n
    if name == "packed":
        base = 4.0 * (n // 32 + 1) + 4.0 * A.packed.numel() + 16.0 * n
    jac = base + 8.0 * n + (n if name == "packed" else 17.0 * n)
    for label, fn, by in (
        (f"spmv {name}", lambda: engine.spmm(A, x), base),
        (f"resid {name}", lambda: _lib.call("bamg_residual", A.ref(), _lib.ptr(b), _lib.ptr(x), _lib.ptr(r)), base + 8.0 * n),
        (f"jacobi(b) {name}", lambda: engine.jacobi(A, d, skip, x, b=b), jac),
    ):
        ms = timed(fn)
        print(f"{label:22s} {ms * 1e3:8.1f} us  {by / 1e6:8.1f} MB  {by / ms / 1e6:8.1f} GB/s", flush=True)
