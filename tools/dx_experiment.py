"""Device time of the input-gradient path (fused dX GEMM, or the unfused
GEMM + combine) at a few short-K shapes (dev tool).

    python tools/dx_experiment.py LABEL [lut|exact] [LUT_SIZE]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw  # noqa: E402

dev = torch.device("cuda", 0)
for (b, i, o, d) in [(16384, 256, 256, 3), (16384, 512, 512, 5), (16384, 256, 256, 8), (32000, 512, 512, 15),
                     (16384, 1024, 1024, 8)]:
    x = torch.rand(b, i, device=dev) * 3 - 1.5
    c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
    dy = torch.randn(b, o, device=dev)
    mode = sys.argv[2] if len(sys.argv) > 2 else "lut"
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
    lut = (ck.exact_basis(ck.BasisKind.CHEBYSHEV, d, device=dev) if mode == "exact"
           else ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=dev))
    prep = PreparedCoeff(c)
    for _ in range(3):
        backward_raw(x, dy, prep, lut, True, want_dc=False, want_db=False)
    torch.cuda.synchronize()
    _lib.timing_collect()
    _lib.timing_enable(True)
    for _ in range(10):
        backward_raw(x, dy, prep, lut, True, want_dc=False, want_db=False)
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    tot = sum(v[0] for k, v in kt.items() if k in ("gemm_dx", "dx_combine")) / 10 * 1e3
    print(sys.argv[1] if len(sys.argv) > 1 else "", (b, i, o, d), "dX path us", round(tot, 1),
          {k: round(v[0] / 10 * 1e3, 1) for k, v in kt.items() if v[1]})
