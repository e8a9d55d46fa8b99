"""GPU parity at the shapes the bench and the sweep report.

The oracle (float64 NumPy restatement of kernels.py:351-447, pinned to the
reference's own outputs by tests/test_oracle_golden.py) runs on a row slice
of each reported configuration -- the full I, O, degree and LUT size -- and
the CUDA path must match it within the normwise tolerance of
tests/test_gpu_parity.py (1e-4 for y, dX, dC; db is a float64 sum).  The
internal chunk size (ck_set_chunk_rows) is lowered so that the chunked dC
accumulation of the wide layers (8 chunks at C4) runs on the slice.  At the
full C4 size (262144 rows) the checks are size-independent: the rows of the
slice inside the full batch match the oracle, dC is linear over the two
halves of the batch, and db is the exact column sum.
"""
import functools

import numpy as np
import pytest
import torch

from oracle import chebykan_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-4

if torch.cuda.is_available():
    import paper_2511_14852_b200 as ck


def _dev():
    return torch.device("cuda", 0)


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=_dev())


@functools.lru_cache(maxsize=None)
def _oracle(b, i, o, d, n, seed):
    """Seeded inputs (perf.py:157-169 distributions) and the oracle's outputs."""
    x, c_jod, dy = orc.bench_inputs(b, i, o, d, seed=seed)
    vals, slopes, _ = orc.build_table(d, n)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    threads = orc.default_threads()
    y = orc.layer_forward(x, c_doj, vals, threads=threads)
    dc, dx, db = orc.layer_backward(x, c_doj, dy, vals, slopes, threads=threads)
    return x, c_doj.astype(np.float32), dy, y, dc, dx, db


def _gpu_layer(x, c_doj, dy, d, n, chunk=None):
    """Through the autograd module (basis cache forward -> backward)."""
    i, o = x.shape[1], dy.shape[1]
    layer = ck.ChebyKANLayer(i, o, d, lut_size=n).to(_dev())
    with torch.no_grad():
        layer.coeff_doj.copy_(_t(c_doj))
    xt = _t(x).requires_grad_(True)
    if chunk is None:
        y = layer(xt)
        y.backward(_t(dy))
    else:
        with ck.chunk_rows(chunk):
            y = layer(xt)
            y.backward(_t(dy))
    torch.cuda.synchronize()
    return (y.detach().cpu().numpy(), layer.coeff_doj.grad.cpu().numpy(), xt.grad.cpu().numpy(),
            layer.bias.grad.cpu().numpy())


def _check(got, want, what):
    y, dc, dx, db = got
    _, _, _, wy, wdc, wdx, wdb = want
    errs = {"y": orc.normwise_err(y, wy), "dC": orc.normwise_err(dc, wdc), "dX": orc.normwise_err(dx, wdx)}
    print(what, {k: f"{v:.2e}" for k, v in errs.items()})
    for k, e in errs.items():
        assert e <= TOL, (what, k, e)
    assert orc.normwise_err(db, wdb) <= 1e-6, what


# C4: 4096 -> 4096, degree 8, N = 32768 (the bench layer)
C4 = (256, 4096, 4096, 8, 32768, 3)


@pytest.mark.parametrize("chunk", [None, 32], ids=["one-chunk", "8-chunks"])
def test_c4_layer_slice_vs_oracle(chunk):
    want = _oracle(*C4)
    x, c, dy = want[:3]
    got = _gpu_layer(x, c, dy, C4[3], C4[4], chunk)
    _check(got, want, f"C4 slice chunk={chunk}")


def test_c4_chunked_dc_equals_one_chunk_dc():
    # the 8-chunk accumulation (ascending order) and the one-chunk GEMM agree
    # to float32 round-off; repeated chunked runs are bitwise identical
    x, c, dy = _oracle(*C4)[:3]
    one = _gpu_layer(x, c, dy, C4[3], C4[4])
    eight = _gpu_layer(x, c, dy, C4[3], C4[4], 32)
    again = _gpu_layer(x, c, dy, C4[3], C4[4], 32)
    assert orc.normwise_err(eight[1], one[1]) <= 1e-5
    for a, b in zip(eight, again):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("shape", [
    (512, 2048, 2048, 5, 32768, 5),    # C1 2048^2 d5
    (256, 4096, 4096, 3, 32768, 6),    # C1 4096^2 d3
    (16384, 256, 256, 3, 32768, 7),    # C1 256^2 d3 at the sweep's full batch (split-R dC, gen forward off)
    (4096, 512, 512, 5, 32768, 8),     # C1 512^2 d5 / C2 hidden layer
    (16384, 64, 512, 5, 32768, 9),     # C2 first layer, full batch
    (16384, 512, 1, 5, 32768, 10),     # C2 head (skinny CUDA-core path), full batch
    (2048, 257, 512, 15, 32768, 11),   # C3 first layer (ragged I)
    (2048, 512, 512, 15, 32768, 12),   # C3 hidden layer
    (2048, 512, 257, 15, 32768, 13),   # C3 output layer (ragged O, transposed dC)
    (128, 40, 256, 8, 32768, 14),      # paper configs (perf.py:137-143): few rows, reduction
    (64, 256, 512, 15, 32768, 15),     # splits across the (segment, K chunk) space
    (32, 512, 1024, 24, 32768, 16),    # d = 24: unfused dX
], ids=lambda s: "x".join(map(str, s[:4])))
def test_reported_shapes_vs_oracle(shape):
    want = _oracle(*shape)
    x, c, dy = want[:3]
    _check(_gpu_layer(x, c, dy, shape[3], shape[4]), want, f"shape {shape[:4]}")


@pytest.mark.parametrize("shape", [(2048, 512, 512, 5, 32768, 8), (2048, 512, 257, 15, 32768, 13)],
                         ids=["512x512d5", "512x257d15"])
def test_reported_shapes_multichunk(shape):
    # the same layers with 300-row chunks (7 chunks, ragged last one)
    want = _oracle(*shape)
    x, c, dy = want[:3]
    _check(_gpu_layer(x, c, dy, shape[3], shape[4], 300), want, f"shape {shape[:4]} chunk=300")


def test_c4_full_batch_properties():
    """The bench configuration itself: 262144 rows x 4096 -> 4096, d8,
    default 32768-row chunks.  Rows 0..255 are the oracle slice of C4."""
    b_full = 262144
    x0, c, dy0, wy, wdc, wdx, wdb = _oracle(*C4)
    dev = _dev()
    g = torch.Generator(device=dev).manual_seed(99)
    x = torch.rand(b_full, 4096, device=dev, generator=g) * 3 - 1.5
    dy = torch.randn(b_full, 4096, device=dev, generator=g)
    x[:256] = _t(x0)
    dy[:256] = _t(dy0)
    layer = ck.ChebyKANLayer(4096, 4096, 8, lut_size=32768).to(dev)
    with torch.no_grad():
        layer.coeff_doj.copy_(_t(c))
    xr = x.requires_grad_(True)
    y = layer(xr)
    y.backward(dy)
    # row independence: the slice's rows inside the full batch vs the oracle
    assert orc.normwise_err(y[:256].detach().cpu().numpy(), wy) <= TOL
    assert orc.normwise_err(xr.grad[:256].cpu().numpy(), wdx) <= TOL
    dc_full = layer.coeff_doj.grad.clone()
    db_full = layer.bias.grad.clone()
    del y
    xr.grad = None
    # linearity over the batch: dC(all rows) = dC(first half) + dC(second half)
    halves = []
    for lo, hi in ((0, b_full // 2), (b_full // 2, b_full)):
        layer.coeff_doj.grad = None
        layer.bias.grad = None
        layer(x[lo:hi].detach()).backward(dy[lo:hi])
        halves.append(layer.coeff_doj.grad.clone())
    err = (dc_full - (halves[0] + halves[1])).abs().max() / dc_full.abs().max()
    print("C4 full: dC linearity", f"{float(err):.2e}")
    assert float(err) <= 1e-5
    # db: float64 column sums
    want_db = dy.double().sum(0)
    assert float((db_full.double() - want_db).abs().max() / want_db.abs().max()) <= 1e-6


def test_c4_full_batch_rank1_dc():
    """dC at the full bench batch (262144 rows = 8 accumulated 32768-row
    chunks) for a rank-1 dy[b, o] = u[b]: every output row of dC equals
    sum_b u_b B_k(x_bi), a matrix-vector product computed here in float64
    from the expansion kernel's basis values (ck_expand, pinned to the
    reference's interp_rows by test_expand_matches_reference_interp)."""
    b_full, chunk = 262144, 32768
    dev = _dev()
    g = torch.Generator(device=dev).manual_seed(123)
    x = torch.rand(b_full, 4096, device=dev, generator=g) * 3 - 1.5
    u = torch.randn(b_full, device=dev, generator=g)
    layer = ck.ChebyKANLayer(4096, 4096, 8, lut_size=32768).to(dev)
    layer(x).backward(u[:, None].expand(b_full, 4096).contiguous())
    dc = layer.coeff_doj.grad  # [9, 4096, 4096]
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, 8, 32768, device=dev)
    ref = torch.zeros(9, 4096, dtype=torch.float64, device=dev)
    for r0 in range(0, b_full, chunk):
        phi = ck.expand(x[r0:r0 + chunk], table)  # [rows, 4096, 9] fp32
        ref += torch.einsum("b,bik->ki", u[r0:r0 + chunk].double(), phi.double())
        del phi
    err = float((dc.double() - ref[:, None, :]).abs().amax() / ref.abs().amax())
    spread = float((dc - dc[:, :1, :]).abs().amax() / dc.abs().amax())
    print("C4 full batch rank-1 dC", f"{err:.2e}", "row spread", f"{spread:.2e}")
    assert err <= TOL
    assert spread <= 1e-6  # every output row of dC is the same reduction
