"""Per-CTA timeline of one tensor-core GEMM launch (dev tool; needs a
library built with -DCK_GEMM_TRACE, e.g. tools/build_variant.py
lib/variants/trace.so -DCK_GEMM_TRACE, then CK_LIB_PATH=...).

    python tools/gemm_trace.py B I O degree [fwd|dx|dc]

Events (us after the earliest kernel entry): 0 entry, 1 prologue barrier
done, 2 griddepcontrol.wait done, 3 first stage landed (MMA warp, leader),
4 last MMA committed (leader), 5 first accumulator drained (epilogue warp 4),
6 epilogue done (warp 4), 7 exit barrier passed.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402
from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw  # noqa: E402

dev = torch.device("cuda", 0)
b, i, o, d = (int(a) for a in sys.argv[1:5])
which = sys.argv[5] if len(sys.argv) > 5 else "fwd"
x = torch.rand(b, i, device=dev) * 3 - 1.5
c = (torch.rand(d + 1, o, i, device=dev) * 2 - 1) / (i * (d + 1)) ** 0.5
dy = torch.randn(b, o, device=dev)
lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 32768, device=dev)
prep = PreparedCoeff(c)
cache = torch.empty(ck.kernels.basis_cache_bytes(b, i, o, d + 1), dtype=torch.uint8, device=dev)
lib = _lib.lib()
fn = lib.ck_debug_gemm_trace
buf = np.zeros((512, 8), dtype=np.uint64)
for rep in range(4):
    forward_raw(x, prep, lut, None, cache)
    if which == "dx":
        backward_raw(x, dy, prep, lut, True, want_dc=False, want_db=False, cache=cache)
    elif which == "dc":
        backward_raw(x, dy, prep, lut, True, want_dx=False, want_db=False, cache=cache)
    torch.cuda.synchronize()
n = fn(buf.ctypes.data, 512)
assert n > 0, "library built without CK_GEMM_TRACE"
t = buf[:n].astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["entry", "prologue", "pdl_wait", "first_stage", "last_mma", "first_acc", "epi_done", "exit"]
print(f"{which} last GEMM launch: {len(t)} CTAs")
for k, nm in enumerate(names):
    col = rel[:, k]
    col = col[t[:, k] > 0]
    if len(col):
        print(f"  {k} {nm:12s} min {col.min():8.2f}  med {np.median(col):8.2f}  max {col.max():8.2f} us  (n={len(col)})")
