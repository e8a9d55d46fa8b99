"""LUT size vs interpolation error against the exact cos(k acos t) path.

CPU-only report (uses the oracle as the measuring instrument): for each
degree and table size, the closed-form bound step^2/8 * k^2(k^2-1)/3
(lut.py:143-153) and the measured max |LUT interp - exact| over a dense grid,
plus the smem footprint a float32 table would need.  Writes markdown to stdout.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import chebykan_oracle as orc

t = np.linspace(-1.0, 1.0, 200_001)
print("| degree | N (lut_size) | bound max_k | measured max_k | float32 table (values) | within 1e-4 budget |")
print("|---|---|---|---|---|---|")
for d in (3, 4, 5, 8, 15):
    exact = orc.chebyshev_trig_rows(d, t)
    for n in (512, 1024, 2048, 4096, 8192, 32768):
        vals, _, _ = orc.build_table(d, n)
        err = np.abs(orc.lut_values(t, vals).T - exact).max(axis=1).max()
        bound = orc.interp_error_bound(d, n).max()
        kib = (d + 1) * n * 4 / 1024
        print(f"| {d} | {n} | {bound:.2e} | {err:.2e} | {kib:.0f} KiB | {'yes' if bound <= 1e-4 else 'no'} |")
