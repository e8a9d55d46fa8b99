"""Markdown table of the key ncu counters per kernel of a report (dev tool).

    python tools/ncu_summary.py REPORT.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor active %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %")]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
cols = [(hdr.index(k), name, units[hdr.index(k)]) for k, name in KEYS if k in hdr]
print("| kernel | " + " | ".join(f"{n} ({u})" for _, n, u in cols) + " |")
print("|---" * (len(cols) + 1) + "|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "")[:60]
    print(f"| `{name}` | " + " | ".join(r[i] for i, _, _ in cols) + " |")
