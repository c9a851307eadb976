"""Histogram of the GEMM shapes one config's setup+solve issues (BAMG_GEMM_LOG lines on stdin)."""
import collections
import sys

c = collections.Counter()
for line in sys.stdin:
    if line.startswith("gemm "):
        c[tuple(int(v) for v in line.split()[1:])] += 1
fl = {s: 2.0 * s[2] * s[3] * s[4] * cnt for s, cnt in c.items()}
print(f"{sum(c.values())} calls, {sum(fl.values()) / 1e12:.2f} TFLOP")
for s, cnt in sorted(c.items(), key=lambda kv: -fl[kv[0]])[:40]:
    print(f"ta={s[0]} tb={s[1]} m={s[2]:6d} n={s[3]:6d} k={s[4]:6d}  x{cnt:5d}  {fl[s] / 1e9:9.1f} GFLOP")
print("by count:")
for s, cnt in c.most_common(15):
    print(f"ta={s[0]} tb={s[1]} m={s[2]:6d} n={s[3]:6d} k={s[4]:6d}  x{cnt:5d}")
