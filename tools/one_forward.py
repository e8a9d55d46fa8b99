import sys, torch
sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck
from paper_2511_14852_b200.kernels import PreparedCoeff, forward_raw
dev = torch.device("cuda", 0)
b, i, o, d = (int(a) for a in sys.argv[1:5])
x = torch.rand(b, i, device=dev) * 3 - 1.5
c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
prep = PreparedCoeff(c)
cache = torch.empty(ck.kernels.basis_cache_bytes(b, i, o, d + 1), dtype=torch.uint8, device=dev)
for _ in range(4):
    forward_raw(x, prep, lut, None, cache)
torch.cuda.synchronize()
