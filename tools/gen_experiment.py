"""Forward with the basis generated in shared memory vs the materialised
planes path (CK_GEN_MAX_O=0), same inputs (dev tool).

    CK_GEN_MAX_O=0 python tools/gen_experiment.py save DIR
    python tools/gen_experiment.py compare DIR
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, forward_raw  # noqa: E402

dev = torch.device("cuda", 0)
mode, out = sys.argv[1], sys.argv[2]
os.makedirs(out, exist_ok=True)
shapes = [(16384, 256, 256, 3), (16384, 256, 256, 5), (16384, 256, 256, 8), (16384, 512, 256, 4),
          (16384, 1024, 256, 8), (16384, 256, 128, 3), (16384, 257, 200, 16), (65536, 256, 256, 3),
          (16384, 64, 256, 1), (16384, 4096, 256, 8), (1000, 100, 60, 7), (16384, 512, 512, 5)]
if os.environ.get("GEN_WIDE"):
    # the wide layers of C1 / C4 (16 and 8 N tiles)
    shapes = [(16384, 4096, 4096, 8), (16384, 2048, 2048, 5), (16384, 4096, 4096, 3), (16384, 1024, 1024, 8)]
if os.environ.get("GEN_NETS"):
    # the C2 / C3 net layers (2 N tiles for the 512-wide outputs)
    shapes = [(16384, 64, 512, 5), (16384, 512, 512, 5), (32000, 257, 512, 15), (32000, 512, 512, 15),
              (32000, 512, 257, 15), (16384, 256, 256, 3), (16384, 512, 512, 3)]
for (b, i, o, d) in shapes:
    g = torch.Generator(device="cpu").manual_seed(b + i + o + d)
    x = (torch.rand(b, i, generator=g) * 3 - 1.5).to(dev)
    c = ((torch.rand(d + 1, o, i, generator=g) * 2 - 1) / (i * (d + 1)) ** 0.5).to(dev)
    bias = torch.randn(o, generator=g).to(dev)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
    prep = PreparedCoeff(c)
    for _ in range(3):
        y = forward_raw(x, prep, lut, bias)
    torch.cuda.synchronize()
    # device time of the library's kernels (per-class CUDA-event timers): the
    # host loop is launch-bound at these sizes
    reps = 20
    _lib.timing_collect()
    _lib.timing_enable(True)
    for _ in range(reps):
        forward_raw(x, prep, lut, bias)
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    us = sum(v[0] for v in kt.values()) / reps * 1e3
    f = os.path.join(out, f"{b}_{i}_{o}_{d}.npy")
    yn = y.cpu().numpy()
    msg = f"{mode} {(b, i, o, d)} fwd {us:.1f} us"
    if mode == "save":
        np.save(f, yn)
    else:
        ref = np.load(f)
        nw = np.linalg.norm(yn - ref) / np.linalg.norm(ref)
        mx = np.max(np.abs(yn - ref)) / np.max(np.abs(ref))
        msg += f"  vs planes: normwise {nw:.2e} max/max {mx:.2e}"
    print(msg, flush=True)
