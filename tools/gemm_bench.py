"""fp64 GEMM throughput: the engine's DMMA kernels (bamg_dgemm) vs torch (cuBLAS).

python tools/gemm_bench.py   -> one line per shape: ms and TFLOP/s of both."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1402_4005_b200 import _lib

SHAPES = [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (16384, 16384, 1024),
          (8192, 8192, 1024), (16384, 28, 16384), (28, 28, 16384), (16384, 1, 16384), (4096, 4096, 64),
          (16384, 16384, 64)]


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for m, n, k in SHAPES:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda")  # column-major m x k
    B = torch.randn(n, k, dtype=torch.float64, device="cuda")  # column-major k x n
    C = torch.zeros(n, m, dtype=torch.float64, device="cuda")
    ours = t(lambda: _lib.call("bamg_dgemm", 0, 0, m, n, k, 1.0, _lib.ptr(A), m, _lib.ptr(B), k, 0.0, _lib.ptr(C), m))
    Am, Bm = A.T, B.T
    ref = t(lambda: torch.matmul(Am, Bm))
    fl = 2.0 * m * n * k
    err = (C.T - Am @ Bm).abs().max().item() / max((Am.abs() @ Bm.abs()).max().item(), 1e-300)
    print(f"{m:6d} {n:6d} {k:6d}  ours {ours:9.3f} ms {fl / ours / 1e9:7.2f} TF/s   cublas {ref:9.3f} ms "
          f"{fl / ref / 1e9:7.2f} TF/s   err {err:.1e}", flush=True)
