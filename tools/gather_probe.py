"""Is the k-wide sweep bound by its gathers or by its own structure? (development tool)

Times the k = 16 SpMM / Jacobi on cfg4's level-0 B and on two synthetic operators with the
same rowptr / values: `self` (every entry's column = its row: all gathers hit L1) and
`near` (columns row-2..row+2: all gathers inside the CTA's tile)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_1402_4005_b200 import engine
from paper_1402_4005_b200.device import DeviceCSR

prob = bench.build_problem("cfg4")
A = DeviceCSR.from_host(prob.B)
n, nnz, k = A.shape[0], A.nnz, 16
rows = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int32),
                               (A.rowptr[1:] - A.rowptr[:-1]).to(torch.int64))
pos = torch.arange(nnz, device="cuda", dtype=torch.int32) - A.rowptr[:-1].to(torch.int64)[rows.long()].to(torch.int32)
ops = {"B": A,
       "self": DeviceCSR(A.rowptr, rows.contiguous(), A.val, A.shape),
       "near": DeviceCSR(A.rowptr, torch.clamp(rows + pos - 2, 0, n - 1).to(torch.int32).contiguous(), A.val, A.shape)}
d = engine.diag(A)
skip = engine.degenerate_rows(A, d)
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.rand((n, k), dtype=torch.float64, device="cuda", generator=g)


def timed(fn, reps=8):
    ts = []
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts[2:])[len(ts[2:]) // 2]


for name, M in ops.items():
    t1 = timed(lambda: engine.spmm(M, X))
    t2 = timed(lambda: engine.jacobi(M, d, skip, X))
    print(f"{name:5s} spmm {t1 * 1e3:8.1f} us   jacobi(hom) {t2 * 1e3:8.1f} us", flush=True)
