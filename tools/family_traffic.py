"""DRAM traffic per launch of the CSR row-kernel family over one bench step.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:"csr_rows_kernel|csr_tile_kernel|rayleigh_fused_kernel" --csv --log-file t.csv \
      python tools/steptimes.py --steps 1
  python tools/family_traffic.py t.csv profiles/r01_csr_family_traffic.json

bench.py reports the result as roofline.traffic (the roofline's kernel family).
"""
import csv
import json
import sys
from collections import defaultdict

path, out = sys.argv[1], sys.argv[2]
alg = None
if len(sys.argv) > 3:  # steptimes --prof output of the same (graph-free) run: algorithmic bytes
    for line in open(sys.argv[3]):
        if line.startswith('{"family": "csr'):
            alg = json.loads(line)
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ii, mi, vi, ui = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    per[r[ii]][r[mi]] = v
n = len(per)
rd = sum(d.get("dram__bytes_read.sum", 0) for d in per.values())
wr = sum(d.get("dram__bytes_write.sum", 0) for d in per.values())
t = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
res = {"family": "csr_stream_spmv_spmm_jacobi", "launches": n, "dram_bytes_per_launch": (rd + wr) / max(n, 1),
       "alg_bytes_per_launch": (alg["alg_bytes"] / max(alg["launches"], 1)) if alg else None,
       "traffic_over_alg": ((rd + wr) / alg["alg_bytes"]) if alg and alg["launches"] == n else None,
       "dram_read_bytes": rd, "dram_write_bytes": wr, "ncu_time_s": t,
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one cfg1 step ({path})"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
