"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0.0, 0])
    total = 0.0
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        name = r[ki].split("(")[0]
        agg[name][0] += us
        agg[name][1] += 1
        total += us
    lines = [f"# ncu launch list summary ({path})", "",
             "Cold-cache, serialised per-launch device times (compare shares, not absolutes).", "",
             f"Total: {total / 1e3:.2f} ms over {sum(c for _, c in agg.values())} launches", "",
             "| kernel | total ms | launches | share |", "|---|---:|---:|---:|"]
    for name, (us, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| `{name}` | {us / 1e3:.3f} | {c} | {100 * us / total:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary ({path})", ""]
    for r in rows[2:]:
        lines.append(f"## `{r[hdr.index('Kernel Name')][:120]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---:|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {r[i]} | {units[i]} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
