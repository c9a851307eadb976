"""Pipeline-bubble finder for one bench step (development tool).

python tools/timeline.py [--config cfg1] [--warmup 3] [--top 30]

Runs bench.py's step (setup + V-cycle operator + GMRES, inputs resident)
`warmup` times, then once with the engine trace on (CUDA events around every
launch, graphs disabled), and reports: step wall time, kernel-busy time, idle
time, the number of host syncs, the largest gaps between consecutive launches
with the kernels either side, and idle time summed by the kernel that precedes
each gap.  The event pairs themselves add ~1-2 us per launch.
"""
import argparse
import ctypes as C
import sys
import time
from collections import defaultdict
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
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--dump", default=None, help="write the ordered launch list (name, start us, duration us) here")
a = ap.parse_args()

name = a.config
fam, size, k, stop, restart, _ = bench.CONFIGS[name]
prob = bench.build_problem(name)
cfg = bench.setup_config(name)
gcfg = pb.GmresConfig(restart=restart, rtol=bench.RTOL)
right, left = bench.draws_for(k, prob.n)
dB = DeviceCSR.from_host(prob.B)
dV = torch.from_numpy(np.ascontiguousarray(right.T)).cuda()
dU = torch.from_numpy(np.ascontiguousarray(left.T)).cuda()
geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda() if prob.geometry is not None else None
P = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
L, c = _lib.lib(), _lib.ctx()


from paper_1402_4005_b200 import bootstrap as bs

marks = []  # (phase, entering, engine launch count)


def rec(name, entering):
    marks.append((name, entering, int(L.bamg_trace_position(c))))


def step():
    setup = pb.run_setup(P, cfg, draws=(dV, dU), B_device=dB)
    rec("vcycle_op", True)
    vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
    rec("vcycle_op", False)
    rec("gmres", True)
    r = pb.gmres(dB, zero, setup.dx0, gcfg, vop, to_host=False)
    rec("gmres", False)
    return r


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
s0, l0 = int(L.bamg_sync_count(c)), int(L.bamg_launch_count(c))
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
wall_plain = (time.perf_counter() - t0) * 1e3
s1, l1 = int(L.bamg_sync_count(c)), int(L.bamg_launch_count(c))
print(f"plain step: {wall_plain:.2f} ms wall, {l1 - l0} launches, {s1 - s0} engine host syncs")

L.bamg_trace_enable(c, 1)
torch.cuda.synchronize()
marks.clear()
bs.RECORDER = rec
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
bs.RECORDER = None
buf = C.create_string_buffer(16 << 20)
L.bamg_trace_timeline(c, buf, 16 << 20)
L.bamg_trace_enable(c, 0)
rows = [r.split("\t") for r in buf.value.decode().splitlines()]
ev = [(r[0], float(r[1]), float(r[2])) for r in rows]
evpos = [int(r[3]) for r in rows]  # trace event index of each entry


if a.dump:
    with open(a.dump, "w") as f:
        for n_, s_, e_ in ev:
            f.write(f"{s_:10.1f}\t{e_ - s_:8.1f}\t{n_}\n")


def marker(name):
    return name.startswith("<") or name.startswith("@")

busy = sum(e - s for n, s, e in ev if not marker(n))
span = ev[-1][2] - ev[0][1]
gaps = []
idle_after = defaultdict(float)
for (pn, ps, pe), (nn, ns, ne) in zip(ev, ev[1:]):
    g = ns - pe
    gaps.append((g, pn, nn, pe))
    idle_after[pn] += g
nsync = sum(1 for n, _, _ in ev if n == "<host sync>")
print(f"traced step: {wall:.2f} ms wall, device span {span / 1e3:.2f} ms, kernel-busy {busy / 1e3:.2f} ms, "
      f"idle {(span - busy) / 1e3:.2f} ms, {len(ev) - nsync} launches, {nsync} engine host syncs")
print(f"gaps > 20 us: {sum(1 for g in gaps if g[0] > 20)} totalling {sum(g[0] for g in gaps if g[0] > 20) / 1e3:.2f} ms")
print("\nlargest gaps (us, after -> before, at us):")
for g, pn, nn, t in sorted(gaps, reverse=True)[:a.top]:
    print(f"{g:9.1f}  {pn[:60]:60s} -> {nn[:50]:50s} @ {t:9.1f}")
print("\nidle summed by preceding launch:")
for n, v in sorted(idle_after.items(), key=lambda kv: -kv[1])[:a.top]:
    print(f"{v / 1e3:8.3f} ms  {n}")

# per phase: launches, kernel-busy, span (from the first launch to the first
# launch after the phase), host syncs
import bisect
stack, spans = [], defaultdict(lambda: [0, 0.0, 0.0, 0])
per_kern = defaultdict(lambda: defaultdict(lambda: [0, 0.0]))
for name, entering, pos in marks:
    if entering:
        stack.append((name, pos))
        continue
    nm, p0 = stack.pop()
    t0 = bisect.bisect_left(evpos, p0)
    t1 = bisect.bisect_left(evpos, pos)
    if t0 >= len(ev) or t1 <= t0:
        continue
    seg = ev[t0:t1]
    sp = spans[nm]
    sp[0] += sum(1 for e in seg if not marker(e[0]))
    sp[1] += sum(e[2] - e[1] for e in seg if not marker(e[0]))
    end = ev[t1][1] if t1 < len(ev) else ev[-1][2]
    sp[2] += end - ev[t0][1]
    sp[3] += sum(1 for e in seg if e[0] == "<host sync>")
    for e in seg:
        if not marker(e[0]):
            pk = per_kern[nm][e[0]]
            pk[0] += 1
            pk[1] += e[2] - e[1]
print("\nper phase (traced): launches, kernel-busy ms, span ms, host syncs")
for nm, (nl, busy_us, span_us, ns) in sorted(spans.items(), key=lambda kv: -kv[1][2]):
    print(f"  {nm:12s} {nl:6d} {busy_us / 1e3:8.2f} {span_us / 1e3:8.2f} {ns:5d}")
for nm, (nl, busy_us, span_us, ns) in sorted(spans.items(), key=lambda kv: -kv[1][2])[:8]:
    print(f"\n[{nm}] top kernels")
    for kn, (cnt, us) in sorted(per_kern[nm].items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"    {us / 1e3:8.3f} ms {cnt:5d}  {kn[:70]}")

# dense coarsest stages (zero-length "@stage" markers at the end of each stage)
st = [(e[0], e[1]) for e in ev if e[0].startswith("@")]
if st:
    print("\ncoarsest stages (ms since previous marker):")
    for (a0, t0), (a1, t1) in zip(st, st[1:]):
        print(f"  {a1[1:]:14s} {(t1 - t0) / 1e3:8.3f}")
