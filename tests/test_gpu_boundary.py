"""Boundary robustness of the C ABI and the module (GPU).

* ck_forward / ck_backward reject a coefficient-prep buffer that is too
  small, was never filled by ck_coeff_prepare, or was prepared for another
  (I, O, K) -- CK_INVALID_ARGUMENT -> ValueError, before any kernel reads it
  (the reference's shape checks, kernels.py:245-260, 395-408).
* ck_coeff_prep_check reads the device header back (validation mode).
* ChebyKANLayer.invalidate_prep() refreshes the bf16 operands after writes
  the autograd version counter does not see (param.data in-place ops).
* Inference (no_grad) never fills a basis cache: narrow layers keep the
  forward that generates the basis in shared memory.
"""
import numpy as np
import pytest
import torch

from oracle import chebykan_oracle as orc

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2511_14852_b200 as ck
    from paper_2511_14852_b200 import _lib
    from paper_2511_14852_b200.kernels import PreparedCoeff


def _dev():
    return torch.device("cuda", 0)


def _fwd(prep_ptr, prep_bytes, x, i, o, lut):
    lib = _lib.lib()
    y = torch.empty(x.shape[0], o, device=_dev())
    ws = torch.empty(max(1, lib.ck_forward_workspace_bytes(x.shape[0], i, o, lut.n_features)), dtype=torch.uint8,
                     device=_dev())
    rc = lib.ck_forward(x.data_ptr(), x.shape[0], i, o, lut.handle, prep_ptr, prep_bytes, None, y.data_ptr(),
                        ws.data_ptr(), ws.numel(), None, 0, _lib.stream_handle(_dev()))
    _lib.check(rc, "ck_forward")
    return y


def _bwd(prep_ptr, prep_bytes, x, dy, i, o, lut):
    lib = _lib.lib()
    dx = torch.empty(x.shape[0], i, device=_dev())
    ws = torch.empty(max(1, lib.ck_backward_workspace_bytes(x.shape[0], i, o, lut.n_features)), dtype=torch.uint8,
                     device=_dev())
    rc = lib.ck_backward(x.data_ptr(), dy.data_ptr(), x.shape[0], i, o, lut.handle, prep_ptr, prep_bytes, 1,
                         dx.data_ptr(), None, None, ws.data_ptr(), ws.numel(), None, 0, None,
                         _lib.stream_handle(_dev()))
    _lib.check(rc, "ck_backward")
    return dx


@pytest.mark.parametrize("o", [48, 2])  # tensor-core layer and skinny layer
def test_prep_buffer_shape_checks(o):
    i, d = 64, 5
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 1024, device=_dev())
    c = torch.randn(d + 1, o, i, device=_dev())
    prep = PreparedCoeff(c)
    x = torch.rand(16, i, device=_dev())
    dy = torch.randn(16, o, device=_dev())
    buf, nbytes = prep.buffer.data_ptr(), prep.buffer.numel()
    _fwd(buf, nbytes, x, i, o, lut)
    _bwd(buf, nbytes, x, dy, i, o, lut)
    prep.check()
    # too small
    with pytest.raises(ValueError, match="coefficient prep buffer too small"):
        _fwd(buf, nbytes - 1, x, i, o, lut)
    # prepared for (64, o, 6), used as (o, 64, 6) / (64, o + 8, 6): same or larger size class
    with pytest.raises(ValueError, match="prepared for"):
        _fwd(buf, 1 << 40, torch.rand(16, o, device=_dev()), o, i, lut)
    with pytest.raises(ValueError, match="prepared for"):
        _bwd(buf, 1 << 40, x, torch.randn(16, o + 8, device=_dev()), i, o + 8, lut)
    with pytest.raises(ValueError, match="prepared for"):
        _lib.check(_lib.lib().ck_coeff_prep_check(buf, 1 << 40, o, i, d + 1), "ck_coeff_prep_check")
    # a damaged device header (the first bytes of the buffer) is caught by the check
    saved = prep.buffer[:16].clone()
    prep.buffer[:4] = 0
    with pytest.raises(ValueError, match="prep header does not match"):
        prep.check()
    prep.buffer[:16] = saved
    prep.check()
    # never prepared
    raw = torch.zeros(nbytes, dtype=torch.uint8, device=_dev())
    with pytest.raises(ValueError, match="not filled by ck_coeff_prepare"):
        _fwd(raw.data_ptr(), nbytes, x, i, o, lut)
    # re-preparing a buffer for another shape moves its record
    c2 = torch.randn(d + 1, o, i + 8, device=_dev())
    big = torch.empty(_lib.lib().ck_coeff_prep_bytes(i + 8, o, d + 1) + nbytes, dtype=torch.uint8, device=_dev())
    for cc, ii in ((c, i), (c2, i + 8)):
        _lib.check(_lib.lib().ck_coeff_prepare(cc.data_ptr(), ii, o, d + 1, big.data_ptr(), big.numel(),
                                               _lib.stream_handle(_dev())), "ck_coeff_prepare")
    with pytest.raises(ValueError, match="prepared for"):
        _fwd(big.data_ptr(), big.numel(), x, i, o, lut)
    _fwd(big.data_ptr(), big.numel(), torch.rand(16, i + 8, device=_dev()), i + 8, o, lut)


def test_invalidate_prep_after_data_write():
    torch.manual_seed(0)
    layer = ck.ChebyKANLayer(96, 64, 4, lut_size=2048).to(_dev())
    x = torch.rand(128, 96, device=_dev()) * 2 - 1
    with torch.no_grad():
        y1 = layer(x)
        layer.coeff_doj.data.mul_(2.0)    # bypasses the version counter
        layer.invalidate_prep()
        y2 = layer(x)
    # scaling by 2 is exact in the bf16 split and in the fp32 accumulation
    assert torch.equal(y2, 2 * y1)
    # in-place on the parameter itself bumps the version: no hook needed
    with torch.no_grad():
        layer.coeff_doj.mul_(0.5)
        y3 = layer(x)
    assert torch.equal(y3, y1)


def test_no_grad_inference_skips_the_basis_cache():
    # 512 -> 256, d5: a narrow layer whose forward generates the basis in
    # shared memory unless a backward wants the planes
    layer = ck.ChebyKANLayer(512, 256, 5, lut_size=32768).to(_dev())
    x = torch.rand(4096, 512, device=_dev()) * 3 - 1.5

    def expand_launches(fn):
        _lib.timing_collect()
        _lib.timing_enable(True)
        out = fn()
        torch.cuda.synchronize()
        _lib.timing_enable(False)
        return out, _lib.timing_collect()["expand"][1]

    with torch.no_grad():
        y_inf, n_inf = expand_launches(lambda: layer(x))
    y_tr, n_tr = expand_launches(lambda: layer(x))
    assert n_inf == 0 and n_tr >= 1
    vals, _, _ = orc.build_table(5, 32768)
    c_doj = layer.coeff_doj.detach().double().cpu().numpy()
    want = orc.layer_forward(x[:256].cpu().numpy(), c_doj, vals, threads=orc.default_threads())
    assert orc.normwise_err(y_inf[:256].cpu().numpy(), want) <= 1e-4
    assert orc.normwise_err(y_tr[:256].detach().cpu().numpy(), want) <= 1e-4
