"""Device time of the skinny-output (d_out <= 8) forward and backward kernels (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw  # noqa: E402

dev = torch.device("cuda", 0)


def dev_us(fn, reps=10):
    _lib.timing_collect()
    _lib.timing_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    return {k: round(v[0] / reps * 1e3, 1) for k, v in kt.items() if v[1]}


for (b, i, o, d) in [(16384, 512, 1, 5), (16384, 512, 4, 3), (65536, 256, 1, 8)]:
    x = torch.rand(b, i, device=dev) * 3 - 1.5
    c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
    dy = torch.randn(b, o, device=dev)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
    prep = PreparedCoeff(c)
    for _ in range(3):
        forward_raw(x, prep, lut, None)
        backward_raw(x, dy, prep, lut, True)
    torch.cuda.synchronize()
    f = dev_us(lambda: forward_raw(x, prep, lut, None))
    g = dev_us(lambda: backward_raw(x, dy, prep, lut, True))
    hbm_f = b * i * 4 / 6.5e12 * 1e6
    print((b, i, o, d), "fwd us", f, "bwd us", g, f"(x read alone at 6.5 TB/s: {hbm_f:.1f} us)", flush=True)
