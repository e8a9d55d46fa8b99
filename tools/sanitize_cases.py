"""Small invocations of every kernel family for compute-sanitizer (dev tool).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases: gemm (expand + the tcgen05 store / dX / dC GEMMs, ragged shapes,
multi-chunk), gen (the forward generating the basis in shared memory),
skinny (d_out <= 8 CUDA-core kernels), partial (forward_partial + combine),
adam (multi-tensor), peer (ck_allreduce_peers / _flags with one rank).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_14852_b200 as ck  # noqa: E402
from paper_2511_14852_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)


def layer_step(b, i, o, d, n=1024, chunk=0):
    layer = ck.ChebyKANLayer(i, o, d, lut_size=n).to(dev)
    x = (torch.rand(b, i, device=dev) * 3 - 1.5).requires_grad_(True)
    with ck.chunk_rows(chunk):
        y = layer(x)
        y.backward(torch.randn_like(y))
    torch.cuda.synchronize()


def case_gemm():
    layer_step(300, 257, 130, 3)            # ragged, transposed dC
    layer_step(600, 96, 300, 5, chunk=256)  # 3 chunks, split-R, segmented store epilogue
    layer_step(256, 64, 64, 17)             # unfused dX (d > 16)


def case_gen():
    layer = ck.ChebyKANLayer(384, 200, 5, lut_size=4096).to(dev)
    with torch.no_grad():
        layer(torch.rand(700, 384, device=dev) * 3 - 1.5)
    torch.cuda.synchronize()


def case_skinny():
    layer_step(500, 257, 1, 5)
    layer_step(300, 64, 5, 3)


def case_partial():
    sched = ck.TileSchedule.for_dims(70, 40, 16, 32)
    c = ck.CoeffTensor(70, 40, 4, ck.Layout.DOJ, torch.randn(5, 40, 70, device=dev))
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, 4, 1024, device=dev)
    buf = ck.PartialBuffer.allocate(sched, 33, instrument=True, device=dev)
    ck.forward_partial(torch.rand(33, 70, device=dev), c, lut, sched, ck.LUT_MODE, buf)
    ck.combine(buf, sched)
    torch.cuda.synchronize()


def case_short():
    # TMA-store epilogue (<= 256 K chunks, 16-byte pitches): forward with
    # bias, split-R partial planes, multi-chunk dC with bulk reduce-add
    layer_step(600, 96, 300, 5, chunk=256)
    layer_step(512, 64, 512, 5)
    layer_step(4000, 64, 256, 3, chunk=1024)


def case_mse():
    for n in (1, 7, 4099, 1 << 20):
        p = torch.randn(n, device=dev, requires_grad=True)
        t = torch.randn(n, device=dev)
        (2.0 * ck.mse(p, t)).backward()
    torch.cuda.synchronize()


def case_adam():
    ps = [torch.nn.Parameter(torch.randn(n, device=dev)) for n in (1, 0, 5, 4099, 70000)]
    for p in ps:
        p.grad = torch.randn_like(p)
    opt = ck.Adam(ps, lr=1e-3)
    opt.step()
    torch.cuda.synchronize()


def case_peer():
    import ctypes

    buf = torch.randn(10001 + 64, device=dev)
    flags = torch.zeros(ck.parallel._lib.lib().ck_peer_flag_words(), dtype=torch.int64, device=dev)
    bufs = (ctypes.c_void_p * 1)(buf.data_ptr())
    fl = (ctypes.c_void_p * 1)(flags.data_ptr())
    lib = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.ck_allreduce_peers(bufs, 1, 0, 10001, s), "peers")
    _lib.check(lib.ck_allreduce_peers_flags(bufs, fl, 1, 0, 0, 10000, 1, 0, s), "peers_flags")
    _lib.check(lib.ck_allreduce_peers_flags(bufs, fl, 1, 0, 4, 9000, 2, 4, s), "peers_flags")
    torch.cuda.synchronize()


CASES = {"short": case_short, "mse": case_mse, "gemm": case_gemm, "gen": case_gen, "skinny": case_skinny, "partial": case_partial, "adam": case_adam,
         "peer": case_peer}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("ok", name, flush=True)
