"""Top SASS instructions by warp-stall samples from an ncu report (development aid).

python tools/ncu_hot.py <report.ncu-rep> [kernel-regex] [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--launch-count", "1"]
if kre:
    cmd += ["--kernel-name", f"regex:{kre}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


body = [r for r in rows[rows.index(hdr) + 1:] if len(r) > i_s and num(r[i_s]) is not None]
tot = sum(num(r[i_s]) for r in body)
print(f"total samples {tot:.0f}, instructions {sum(num(r[i_ex]) for r in body):.0f}")
for r in sorted(body, key=lambda r: -num(r[i_s]))[:top]:
    print(f"{num(r[i_s]):7.0f} {100 * num(r[i_s]) / max(tot, 1):5.1f}%  ex={r[i_ex]:>7}  {r[0][-5:]}  {r[i_src].strip()}")
