"""Compare the fused dX of the chord-slope epilogue with the gathered-slope
one (CK_DX_CHORD=0) on the same inputs (dev tool).

    CK_DX_CHORD=0 python tools/chord_check.py save DIR
    python tools/chord_check.py compare DIR
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw  # noqa: E402

dev = torch.device("cuda", 0)
mode, out = sys.argv[1], sys.argv[2]
os.makedirs(out, exist_ok=True)
cases = [(4096, 256, 256, d, kind, n) for d in (1, 3, 5, 8, 12, 16)
         for kind in (ck.BasisKind.CHEBYSHEV, ck.BasisKind.LEGENDRE, ck.BasisKind.HERMITE)
         for n in (32768, 1024)]
for (b, i, o, d, kind, n) in cases:
    g = torch.Generator(device="cpu").manual_seed(d * 100 + n % 97)
    x = (torch.rand(b, i, generator=g) * 6 - 3).to(dev)
    c = ((torch.rand(d + 1, o, i, generator=g) * 2 - 1) / (i * (d + 1)) ** 0.5).to(dev)
    dy = torch.randn(b, o, generator=g).to(dev)
    lut = ck.lut_build(kind, d, n, device=dev)
    dx = backward_raw(x, dy, PreparedCoeff(c), lut, True, want_dc=False, want_db=False)[1].cpu().numpy()
    f = os.path.join(out, f"{kind.value}_{d}_{n}.npy")
    if mode == "save":
        np.save(f, dx)
    else:
        ref = np.load(f)
        nw = np.linalg.norm(dx - ref) / np.linalg.norm(ref)
        mx = np.max(np.abs(dx - ref)) / np.max(np.abs(ref))
        print(f"{kind.value:10s} d={d:2d} N={n:5d} normwise {nw:.2e} max/max {mx:.2e}", flush=True)
