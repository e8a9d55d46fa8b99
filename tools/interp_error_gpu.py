"""LUT size vs interpolation error measured ON THE GPU: the table path
(ck_expand on a LutTable) against the exact path (ck_expand on an exact
handle: cos(k acos t) for Chebyshev, the recurrences for the other families),
on the same float32 inputs, plus the layer-level effect (fused forward, LUT
vs exact, normwise).  Writes markdown to stdout; the float32 evaluation floor
is ~1e-7 * k^2.

    python tools/interp_error_gpu.py > profiles/lut_interp_error_gpu.md
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402

dev = torch.device("cuda", 0)
t = torch.linspace(-0.999, 0.999, 400_001, dtype=torch.float64)
x = torch.atanh(t).to(torch.float32).to(dev).reshape(1, -1)

print("| basis | degree | N | bound max_k (lut_max_error_bound) | GPU measured max_k |LUT - exact| | layer y normwise (LUT vs exact) |")
print("|---|---|---|---|---|---|")
rng = np.random.default_rng(0)
for kind, degrees in ((ck.BasisKind.CHEBYSHEV, (3, 5, 8, 15)), (ck.BasisKind.LEGENDRE, (5, 8)),
                      (ck.BasisKind.HERMITE, (5,)), (ck.BasisKind.FOURIER, (4,))):
    for d in degrees:
        exact = ck.exact_basis(kind, d, device=dev, trig=kind is ck.BasisKind.CHEBYSHEV)
        pe = ck.expand(x, exact)
        k = ck.feature_count(kind, d)
        i, o, b = 256, 128, 2048
        s = 1.0 / np.sqrt(i * k)
        xs = torch.tensor(rng.uniform(-2, 2, (b, i)), dtype=torch.float32, device=dev)
        c = ck.CoeffTensor(i, o, k - 1, ck.Layout.DOJ,
                           torch.tensor(rng.uniform(-s, s, (k, o, i)), dtype=torch.float32, device=dev))
        ye = ck.fused_forward(xs, c, None, None, ck.EXACT_MODE, kind=kind)
        for n in (1024, 4096, 32768):
            lut = ck.lut_build(kind, d, n, device=dev)
            pl = ck.expand(x, lut)
            err = (pl - pe).abs().amax().item()
            bound = float(np.max(ck.lut_max_error_bound(lut)))
            yl = ck.fused_forward(xs, c, lut)
            yn = ((yl - ye).abs().max() / ye.abs().max()).item()
            print(f"| {kind.value} | {d} | {n} | {bound:.2e} | {err:.2e} | {yn:.2e} |", flush=True)
