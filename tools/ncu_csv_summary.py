"""Key ncu counters per kernel from an exported `--page raw --csv` file (dev tool).

    python tools/ncu_csv_summary.py RAW.csv [extra_metric ...]
"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM rd"),
        ("dram__bytes_write.sum", "DRAM wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"),
        ("smsp__inst_executed.sum", "warp inst"),
        ("sm__cycles_elapsed.avg.per_second", "SM clk")]
KEYS += [(k, k) for k in sys.argv[2:]]

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, units = rows[0], rows[1]
cols = [(hdr.index(k), name, units[hdr.index(k)]) for k, name in KEYS if k in hdr]
print("| # | kernel | " + " | ".join(f"{n} ({u})" if u else n for _, n, u in cols) + " |")
print("|---" * (len(cols) + 2) + "|")
for j, r in enumerate(rows[2:]):
    name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "").replace("ck::", "")[:48]
    print(f"| {j} | `{name}` | " + " | ".join(r[i] for i, _, _ in cols) + " |")
