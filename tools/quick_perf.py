"""Quick CUDA-event timing of fused forward / backward at a few shapes (dev tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw

dev = torch.device("cuda", 0)


def bench(b, i, o, d, n=32768, reps=5):
    x = torch.rand(b, i, device=dev) * 3 - 1.5
    s = 1 / np.sqrt(i * (d + 1))
    c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) * s
    dy = torch.randn(b, o, device=dev)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=dev)
    prep = PreparedCoeff(c)
    forward_raw(x, prep, lut, None)
    backward_raw(x, dy, prep, lut, True)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        e[0].record()
        forward_raw(x, prep, lut, None)
        e[1].record()
        backward_raw(x, dy, prep, lut, True)
        e[2].record()
        torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1]))
        tb.append(e[1].elapsed_time(e[2]))
    f = ck.count_flops(b, i, o, d)
    mf, mb = np.median(tf), np.median(tb)
    print(f"B={b} {i}->{o} d{d} N={n}: fwd {mf:.3f} ms ({f['fwd']/mf/1e9:.1f} TF/s alg)  "
          f"bwd {mb:.3f} ms ({f['bwd']/mb/1e9:.1f} TF/s alg)  train {b/(mf+mb)*1e3:.0f} samples/s", flush=True)


if __name__ == "__main__":
    for shp in [(16384, 256, 256, 3), (16384, 1024, 1024, 8), (16384, 4096, 4096, 8), (16384, 2048, 2048, 5)]:
        bench(*shp)
