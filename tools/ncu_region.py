"""Summarise an ncu source page: stall reasons per SASS address region (dev tool).

    python tools/ncu_region.py REPORT KERNEL_REGEX LAUNCH_SKIP [split_addr_hex ...]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
splits = [int(a, 16) for a in sys.argv[4:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1][:100])
h = rows[1]
ai, si, ii = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
names = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
idx = {n: h.index(n) for n in names}
reg = defaultdict(lambda: defaultdict(int))
top = []
seen = set()
for r in rows[2:]:
    try:
        a = int(r[ai], 16) & 0xFFFFF
    except ValueError:
        break
    if a in seen:
        continue
    seen.add(a)
    region = sum(1 for s in splits if a >= s)
    tot = 0
    for n in names:
        v = int(r[idx[n]] or 0)
        reg[region][n] += v
        tot += v
    top.append((tot, a, r[si].strip()[:80], r[ii]))
for region in sorted(reg):
    d = reg[region]
    tot = sum(d.values())
    print(f"region {region}: {tot} samples", {k: v for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:6]})
for t in sorted(top, reverse=True)[:25]:
    print(f"{t[0]:7d} {t[1]:06x} {t[3]:>10s} {t[2]}")
