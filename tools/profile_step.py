"""One training step of a ChebyKAN layer for ncu captures (dev tool).

    python tools/profile_step.py [B I O degree lut_size]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck

args = [int(a) for a in sys.argv[1:]]
b, i, o, d, n = (args + [16384, 4096, 4096, 8, 32768][len(args):])[:5]
dev = torch.device("cuda", 0)
layer = ck.ChebyKANLayer(i, o, d, lut_size=n).to(dev)
x = (torch.rand(b, i, device=dev) * 3 - 1.5).requires_grad_(True)
dy = torch.randn(b, o, device=dev)
for _ in range(2):  # warmup step + profiled step
    x.grad = None
    y = layer(x)
    y.backward(dy)
torch.cuda.synchronize()
print("ok", b, i, o, d, n)
