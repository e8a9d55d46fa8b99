"""Hottest SASS instructions (warp-stall samples) of an ncu report (dev tool).

    python tools/ncu_sass_hot.py REPORT.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ix = {n: i for i, n in enumerate(h)}


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


data = [r for r in rows[1:] if len(r) == len(h)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(num(r[ix[key]]) for r in data) or 1.0
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
print(f"samples {tot:.0f}, instructions {len(data)}")
for r in sorted(data, key=lambda r: -num(r[ix[key]]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    rs = sorted(((k, num(r[ix[k]])) for k in reasons), key=lambda kv: -kv[1])[:3]
    print(f"{num(r[ix[key]]) / tot * 100:5.1f}%  {r[ix['Source']].strip()[:58]:58s} "
          + " ".join(f"{k[6:]}={v:.0f}" for k, v in rs if v))
