"""Stall breakdown and hottest SASS lines per kernel from an exported
`--page source --csv --print-source sass` file (dev tool).

    python tools/ncu_src_stalls.py SRC.csv [kernel_regex] [top_n]
"""
import collections
import csv
import io
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


seen = set()
for b in blocks:
    name = b[0].split(",", 1)[1][:100]
    if pat and not pat.search(name):
        continue
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    data = [r for r in rows[1:] if len(r) == len(h)]
    st = {k: sum(num(r[ix[k]]) for r in data) for k in h if k.startswith("stall_") and "Not Issued" not in k}
    tot = sum(st.values()) or 1.0
    inst = sum(num(r[ix["Instructions Executed"]]) for r in data)
    print(name, f"warp inst {inst:.0f}, stall samples {tot:.0f}")
    print("  ", {k[6:]: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:7]})
    samp = "Warp Stall Sampling (All Samples)"
    for r in sorted(data, key=lambda r: -num(r[ix[samp]]))[:top]:
        print(f"    {num(r[ix[samp]]) / tot * 100:5.1f}%  {r[ix['Source']].strip()[:90]}")
