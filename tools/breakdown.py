"""Per-kernel-class device time of one training step (library CUDA-event timers)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck
from paper_2511_14852_b200 import _lib
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw

dev = torch.device("cuda", 0)
args = [int(a) for a in sys.argv[1:]]
b, i, o, d, n = (args + [16384, 4096, 4096, 8, 32768][len(args):])[:5]
x = torch.rand(b, i, device=dev) * 3 - 1.5
c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
dy = torch.randn(b, o, device=dev)
lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=dev)
prep = PreparedCoeff(c)
for _ in range(2):
    forward_raw(x, prep, lut, None)
    backward_raw(x, dy, prep, lut, True)
torch.cuda.synchronize()
_lib.timing_collect()
_lib.timing_enable(True)
reps = 3
for _ in range(reps):
    forward_raw(x, prep, lut, None)
    backward_raw(x, dy, prep, lut, True)
torch.cuda.synchronize()
try:
    import pynvml
    pynvml.nvmlInit()
    clk = pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
except Exception:
    clk = -1
_lib.timing_enable(False)
kt = _lib.timing_collect()
fl = 2 * b * i * o * d
tot = sum(v[0] for v in kt.values()) / reps
print(f"B={b} {i}->{o} d{d} N={n}: total kernel {tot:.3f} ms/step  (sm clock at end {clk} MHz)")
for k, (ms, cnt) in kt.items():
    if cnt:
        extra = f"  {fl / (ms / reps) / 1e9:7.1f} TF/s alg" if k.startswith("gemm") else ""
        print(f"  {k:10s} {ms / reps:8.3f} ms  {cnt // reps:3d} launches{extra}")
