"""Print an ncu gpu__time_duration launch list as a compact table (dev tool).

    python tools/launch_table.py launches.csv
"""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = 0.0
for r in rows[1:]:
    if r[vi] in ("", "Metric Value"):
        continue
    v = float(r[vi].replace(",", ""))
    us = v / 1000.0 if r[ui] in ("nsecond", "ns") else v if r[ui] in ("usecond", "us") else v * 1000
    tot += us
    name = re.sub(r"\(.*", "", r[ki])[:90]
    print(f"{us:9.2f} us  {name}")
print(f"{tot:9.2f} us  total")
