"""Summarise ncu --csv metric logs of the GEMMs (dev tool).

    python tools/ncu_metrics_table.py gpurun_out/pace_w*.csv
"""
import collections
import csv
import re
import sys


def fl(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def table(path):
    rows = [line for line in open(path) if line.startswith('"')]
    r = list(csv.reader(rows))
    hdr, data = r[0], r[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for d in data:
        m = re.search(r"kernel<([^>]*)>", d[ki])
        per.setdefault((d[ii], m.group(1) if m else d[ki][:40]), {})[d[mi]] = d[vi]
    out = []
    for (_, k), m in per.items():
        g = lambda n: fl(m.get(n, "nan"))  # noqa: E731
        out.append((k, g("gpu__time_duration.sum") / 1e6, g("dram__bytes_read.sum") / 1e9,
                    g("dram__bytes_write.sum") / 1e9, g("lts__t_sectors_srcunit_tex_op_read.sum") * 32 / 1e9,
                    g("lts__t_sector_op_read_hit_rate.pct"), g("sm__cycles_elapsed.avg.per_second") / 1e9))
    return out


if __name__ == "__main__":
    print("| capture | kernel | time (ms) | DRAM read (GB) | DRAM write (GB) | L2 read (GB) | L2 hit % | SM clock (GHz) |")
    print("|---|---|---|---|---|---|---|---|")
    for p in sys.argv[1:]:
        for k, t, dr, dw, l2, hit, clk in table(p):
            print(f"| {p.split('/')[-1]} | `{k}` | {t:.2f} | {dr:.1f} | {dw:.2f} | {l2:.1f} | {hit:.1f} | {clk:.3f} |")
