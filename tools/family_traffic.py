"""DRAM traffic per launch of the roofline's kernel families over one bench step.

  BAMG_NO_GRAPHS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:"csr_rows|rayleigh_fused_kernel|cgs_dots_kernel|cgs_final_kernel|cgs_update" --csv --log-file t.csv \
      python tools/steptimes.py --config cfg4 --steps 1 --prof > alg.txt
  python tools/family_traffic.py t.csv alg.txt profiles/r02_family_traffic.json cfg4

Graph-free run (every launch profiled and event-timed), so ncu's DRAM bytes and
the engine's algorithmic bytes cover the same launches.  bench.py reports
roofline.traffic as (DRAM / algorithmic) of its dominant family applied per
launch.
"""
import csv
import json
import re
import sys
from collections import defaultdict

FAMILIES = {"csr_stream_spmv_spmm_jacobi": r"csr_rows_kernel|csr_rows_pipe_kernel|csr_rows_packed_kernel|csr_rows_stencil_kernel|csr_rows_stencil1_kernel|rayleigh_fused_kernel",
            "gmres_cgs2_basis_passes": r"cgs_dots_kernel|cgs_final_kernel|cgs_update_kernel|cgs_update_pair_kernel"}

path, algp, out = sys.argv[1], sys.argv[2], sys.argv[3]
cfgname = sys.argv[4] if len(sys.argv) > 4 else "cfg4"
alg = {}
for line in open(algp):
    if line.startswith('{"family"'):
        d = json.loads(line)
        alg[d["family"]] = d
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
per = defaultdict(dict)
name = {}
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name[r[ii]] = r[ki]
res = {"config": cfgname, "families": {}}
for fam, rx in FAMILIES.items():
    ids = [i for i in per if re.search(rx, name[i])]
    rd = sum(per[i].get("dram__bytes_read.sum", 0) for i in ids)
    wr = sum(per[i].get("dram__bytes_write.sum", 0) for i in ids)
    t = sum(per[i].get("gpu__time_duration.sum", 0) for i in ids)
    a = alg.get(fam)
    n = len(ids)
    res["families"][fam] = {
        "launches": n, "dram_bytes_per_launch": (rd + wr) / max(n, 1),
        "alg_bytes_per_launch": (a["alg_bytes"] / max(a["launches"], 1)) if a else None,
        "traffic_over_alg": ((rd + wr) / a["alg_bytes"]) if a and a["launches"] == n and a["alg_bytes"] else None,
        "dram_read_bytes": rd, "dram_write_bytes": wr, "ncu_time_s": t,
        "ncu_GBps": (rd + wr) / t / 1e9 if t else None}
res["source"] = f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one graph-free {cfgname} step ({path})"
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
