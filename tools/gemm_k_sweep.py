"""Forward-GEMM device time vs reduction length at a fixed output (dev tool):
separates the per-launch fixed cost from the per-iteration cost of the
short-K tiles.

    python tools/gemm_k_sweep.py [rows] [d_out] [degree]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, forward_raw  # noqa: E402

dev = torch.device("cuda", 0)
b = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
o = int(sys.argv[2]) if len(sys.argv) > 2 else 512
d = int(sys.argv[3]) if len(sys.argv) > 3 else 4
for i in (16, 32, 64, 128, 256, 512, 1024, 2048):
    x = torch.rand(b, i, device=dev) * 3 - 1.5
    c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
    prep = PreparedCoeff(c)
    cache = torch.empty(ck.kernels.basis_cache_bytes(b, i, o, d + 1), dtype=torch.uint8, device=dev)
    for _ in range(3):
        forward_raw(x, prep, lut, None, cache)
    torch.cuda.synchronize()
    reps = 30
    _lib.timing_collect()
    _lib.timing_enable(True)
    for _ in range(reps):
        forward_raw(x, prep, lut, None, cache)
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    its = -(-i * d // 64)
    print(f"rows {b} {i}->{o} d{d}: K chunks {its:4d}  " +
          "  ".join(f"{k} {v[0] / reps * 1e3:7.1f} us" for k, v in kt.items() if v[1]), flush=True)
