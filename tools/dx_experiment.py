import sys, torch
sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw
from paper_2511_14852_b200 import _lib
dev = torch.device("cuda", 0)
for (b, i, o, d) in [(16384, 256, 256, 3), (16384, 512, 512, 5), (16384, 256, 256, 8)]:
    x = torch.rand(b, i, device=dev) * 3 - 1.5
    c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
    dy = torch.randn(b, o, device=dev)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
    prep = PreparedCoeff(c)
    for _ in range(3):
        backward_raw(x, dy, prep, lut, True, want_dc=False, want_db=False)
    torch.cuda.synchronize()
    _lib.timing_collect(); _lib.timing_enable(True)
    for _ in range(10):
        backward_raw(x, dy, prep, lut, True, want_dc=False, want_db=False)
    torch.cuda.synchronize(); _lib.timing_enable(False)
    kt = _lib.timing_collect()
    print(sys.argv[1], (b, i, o, d), "gemm_dx us/launch", round(kt["gemm_dx"][0] / kt["gemm_dx"][1] * 1e3, 1))
