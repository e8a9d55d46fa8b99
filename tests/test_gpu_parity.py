"""GPU parity: the sm_100a kernels through the C ABI vs the reference.

Gates (north star): normwise error max|got-want|/max|want|
<= 1e-4 for y, dX, dC and db against the float64 reference on identical
float32 inputs at the same LUT size; the float64 LUT itself and the cell
slopes are bit-exact; repeated runs are bitwise identical.
"""
import numpy as np
import pytest
import torch

from conftest import golden_kind_cases, golden_kind_lut_cases, golden_layer_cases, golden_lut_cases
from oracle import chebykan_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-4  # normwise, fp32 I/O + BF16x3 tensor-core contractions

if torch.cuda.is_available():
    import paper_2511_14852_b200 as ck
    from paper_2511_14852_b200 import _lib


def _dev():
    return torch.device("cuda", 0)


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=_dev())


def test_device_is_b200_and_library_loads():
    assert torch.cuda.is_available()
    assert _lib.lib().ck_device_supported(0) == 1, torch.cuda.get_device_name(0)


@pytest.mark.parametrize("degree,n", [(2, 3), (8, 1024), (8, 4096), (3, 512), (15, 16384), (5, 32768), (0, 16)])
def test_lut_build_bit_identical_to_oracle(degree, n):
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, degree, n, device=_dev())
    v, s, step = orc.build_table(degree, n)
    assert table.step == step
    assert np.array_equal(table.values, v)
    assert np.array_equal(table.slopes, s)


@pytest.mark.parametrize("path", golden_lut_cases(), ids=lambda p: p.stem)
def test_expand_matches_reference_interp(path):
    g = np.load(path)
    degree = int(path.stem.split("_")[1][1:])
    n = int(path.stem.split("_")[2][1:])
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, degree, n, device=_dev())
    # feed pre-images so the kernel's tanh lands on the reference's points
    t = g["points"].astype(np.float64)
    x = np.arctanh(np.clip(t, -1 + 1e-7, 1 - 1e-7)).astype(np.float32)
    tt = np.tanh(x.astype(np.float64))
    want_v, want_s = orc.lut_values_and_slopes(tt, *orc.build_table(degree, n)[:2])
    phi, slopes = ck.expand(_t(x).reshape(1, -1), table, with_slopes=True)
    phi = phi.reshape(-1, degree + 1).cpu().numpy()
    slopes = slopes.reshape(-1, degree + 1).cpu().numpy()
    assert np.abs(phi - want_v).max() <= 2e-6
    # float64 cell choice: slopes are the reference's float32 table entries
    assert np.array_equal(slopes.astype(np.float64), want_s)


def _run_layer(g):
    degree, n = int(g["degree"]), int(g["lut_size"])
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, degree, n, device=_dev())
    c = ck.reorder_to_doj(ck.CoeffTensor(g["x"].shape[1], g["dy"].shape[1], degree, ck.Layout.JOD,
                                          _t(g["c_jod"])))
    bias = _t(g["bias"]) if "bias" in g else None
    mode = ck.KernelMode(include_tanh_jacobian=bool(g["jacobian"]))
    y = ck.fused_forward(_t(g["x"]), c, table, None, mode, bias)
    cg, dx = ck.backward_fused(_t(g["x"]), c, _t(g["dy"]), table, None, mode)
    return y.cpu().numpy(), cg.data.cpu().numpy(), dx.cpu().numpy()


@pytest.mark.parametrize("path", golden_layer_cases(), ids=lambda p: p.stem)
def test_layer_matches_reference_golden(path):
    g = np.load(path)
    y, dc, dx = _run_layer(g)
    errs = {
        "y": orc.normwise_err(y, g["y"]),
        "dc": orc.normwise_err(dc, g["dc_doj"]),
        "dx": orc.normwise_err(dx, g["dx"]),
    }
    print(path.stem, {k: f"{v:.2e}" for k, v in errs.items()})
    for k, e in errs.items():
        assert e <= TOL, (k, e)


@pytest.mark.parametrize("path", golden_layer_cases(), ids=lambda p: p.stem)
def test_module_autograd_matches_reference_golden(path):
    g = np.load(path)
    degree, n = int(g["degree"]), int(g["lut_size"])
    i, o = g["x"].shape[1], g["dy"].shape[1]
    layer = ck.ChebyKANLayer(i, o, degree, bias="bias" in g, lut_size=n,
                             include_tanh_jacobian=bool(g["jacobian"])).to(_dev())
    layer.load_jod(g["c_jod"])
    if "bias" in g:
        with torch.no_grad():
            layer.bias.copy_(_t(g["bias"]))
    x = _t(g["x"]).requires_grad_(True)
    y = layer(x)
    y.backward(_t(g["dy"]))
    assert orc.normwise_err(y.detach().cpu().numpy(), g["y"]) <= TOL
    assert orc.normwise_err(layer.coeff_doj.grad.cpu().numpy(), g["dc_doj"]) <= TOL
    assert orc.normwise_err(x.grad.cpu().numpy(), g["dx"]) <= TOL
    if "bias" in g:
        assert orc.normwise_err(layer.bias.grad.cpu().numpy(), g["db"]) <= 1e-6


@pytest.mark.parametrize("shape", [(512, 1024, 1024, 8, 32768), (300, 257, 130, 3, 512),
                                   (1024, 64, 64, 4, 4096), (2048, 512, 512, 5, 1024),
                                   (257, 96, 1, 5, 1024), (64, 257, 512, 15, 16384),
                                   (128, 64, 48, 17, 2048), (96, 40, 300, 24, 32768),
                                   # d_out = 257 < d_in: the dC GEMM runs transposed (M = d_in);
                                   # the second one over two 32768-row chunks (accumulated dC)
                                   (700, 512, 257, 3, 1024), (33000, 256, 257, 1, 256)])
def test_random_shapes_vs_oracle(shape):
    b, i, o, d, n = shape
    x, c_jod, dy = orc.bench_inputs(b, i, o, d, seed=b + i + o)
    vals, slopes, _ = orc.build_table(d, n)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    want_y = orc.layer_forward(x, c_doj, vals, threads=8)
    want_dc, want_dx, want_db = orc.layer_backward(x, c_doj, dy, vals, slopes, threads=8)
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=_dev())
    c = ck.CoeffTensor(i, o, d, ck.Layout.DOJ, _t(c_doj.astype(np.float32)))
    y = ck.fused_forward(_t(x), c, table).cpu().numpy()
    cg, dx = ck.backward_fused(_t(x), c, _t(dy), table)
    e = (orc.normwise_err(y, want_y), orc.normwise_err(cg.data.cpu().numpy(), want_dc),
         orc.normwise_err(dx.cpu().numpy(), want_dx))
    print(shape, [f"{v:.2e}" for v in e])
    assert max(e) <= TOL, e


def test_bitwise_determinism():
    b, i, o, d = 4096, 512, 384, 6
    x, c_jod, dy = orc.bench_inputs(b, i, o, d, seed=7)
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, 4096, device=_dev())
    c = ck.reorder_to_doj(ck.CoeffTensor(i, o, d, ck.Layout.JOD, _t(c_jod)))
    outs = []
    for _ in range(3):
        y = ck.fused_forward(_t(x), c, table)
        cg, dx = ck.backward_fused(_t(x), c, _t(dy), table)
        outs.append((y, cg.data, dx))
    for other in outs[1:]:
        for a, bb in zip(outs[0], other):
            assert torch.equal(a, bb)


def test_error_paths_match_reference_wording():
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, 2, 64, device=_dev())
    c_jod = ck.CoeffTensor(3, 2, 2, ck.Layout.JOD, torch.ones(18, device=_dev()))
    with pytest.raises(ValueError, match="DOJ"):
        ck.fused_forward(torch.zeros(1, 3, device=_dev()), c_jod, table)
    c = ck.reorder_to_doj(c_jod)
    with pytest.raises(ValueError, match="input width 4 != coefficient d_in 3"):
        ck.fused_forward(torch.zeros(2, 4, device=_dev()), c, table)
    with pytest.raises(ValueError, match="dy must have shape"):
        ck.backward_fused(torch.zeros(2, 3, device=_dev()), c, torch.zeros(2, 3, device=_dev()), table)
    other = ck.lut_build(ck.BasisKind.CHEBYSHEV, 3, 64, device=_dev())
    with pytest.raises(ValueError, match="LUT has 4 features, coefficients expect 3"):
        ck.fused_forward(torch.zeros(2, 3, device=_dev()), c, other)
    x = torch.zeros(2, 3, device=_dev())
    x[1, 2] = float("inf")
    with pytest.raises(ck.NonFiniteInputError, match=r"b=1, j=2"):
        ck.fused_forward(x, c, table, validate=True)


def test_hand_examples():
    # test_kernels.py:63-70 (LUT mode at N=32768: linear features are exact
    # up to float32): all-ones coefficients, X = [0, 10] -> 1 + (1 + tanh 10)
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, 1, 32768, device=_dev())
    c = ck.CoeffTensor(2, 1, 1, ck.Layout.DOJ, torch.ones(4, device=_dev()))
    y = ck.fused_forward(torch.tensor([[0.0, 10.0]], device=_dev()), c, table)
    assert abs(float(y[0, 0]) - (2.0 + np.tanh(10.0))) <= 1e-6
    # degree 0: dC = sum_b dy for every j, dX = 0 (test_kernels.py:152-162)
    t0 = ck.lut_build(ck.BasisKind.CHEBYSHEV, 0, 16, device=_dev())
    c0 = ck.CoeffTensor(3, 2, 0, ck.Layout.DOJ, torch.ones(6, device=_dev()))
    x = torch.tensor([[0.1, -0.4, 2.0], [1.0, 0.0, -1.0]], device=_dev())
    dy = torch.tensor([[1.0, 2.0], [3.0, 4.0]], device=_dev())
    cg, dx = ck.backward_fused(x, c0, dy, t0)
    assert torch.count_nonzero(dx) == 0
    for j in range(3):
        assert torch.equal(cg.data[0, :, j], dy.sum(0))


@pytest.mark.parametrize("n", [1024, 32768])
def test_dx_cells_exact_at_cell_edges(n):
    # Inputs placed within a few float32 ulps of cell edges (where a float32
    # tanh would pick the neighbouring cell): the fused dX must
    # still use the reference's float64 cell, so no element may show the
    # ~1e-3 relative error a wrong (piecewise-constant) slope produces.
    b, i, o, d = 64, 256, 64, 8
    rng = np.random.default_rng(n)
    step = 2.0 / (n - 1)
    cells = rng.integers(1, n - 1, size=(b, i))
    x = np.arctanh(-1.0 + cells * step).astype(np.float32)
    ulps = rng.integers(-3, 4, size=(b, i)).astype(np.float32)
    x = (x + ulps * np.spacing(x)).astype(np.float32)
    _, c_jod, dy = orc.bench_inputs(b, i, o, d, seed=3)
    vals, slopes, _ = orc.build_table(d, n)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    _, want_dx, _ = orc.layer_backward(x, c_doj, dy, vals, slopes)
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=_dev())
    c = ck.CoeffTensor(i, o, d, ck.Layout.DOJ, _t(c_doj.astype(np.float32)))
    _, dx = ck.backward_fused(_t(x), c, _t(dy), table)
    got = dx.cpu().numpy().astype(np.float64)
    assert orc.normwise_err(got, want_dx) <= TOL
    # elementwise on the elements that carry signal: BF16x3 round-off stays
    # ~1e-5 relative, a wrong cell's slope would show >= ~1e-3
    big = np.abs(want_dx) > 0.05 * np.abs(want_dx).max()
    rel = np.abs(got - want_dx)[big] / np.abs(want_dx)[big]
    assert rel.max() <= 5e-4, (rel.max(), int((rel > 5e-4).sum()))


# ---------------------------------------------------------------------------
# Other basis families (LUT mode) and the exact-evaluation path


@pytest.mark.parametrize("path", golden_kind_lut_cases(), ids=lambda p: p.stem)
def test_kind_lut_build_matches_reference(path):
    g = np.load(path)
    kind, degree, n = str(g["kind"]), int(g["degree"]), int(g["lut_size"])
    table = ck.lut_build(ck.BasisKind(kind), degree, n, device=_dev())
    assert table.n_features == orc.feature_count(kind, degree)
    v, s = table.values, table.slopes
    cols = g["cols"]
    if kind == "fourier":
        # cos/sin(pi x) come from the host libm like numpy's; allow 2 ulp in
        # case the GPU box's numpy dispatches another float64 cos/sin
        np.testing.assert_allclose(v[:, cols], g["values"], rtol=0, atol=5e-16)
        assert np.abs(s[:, cols[cols < n - 1]].astype(np.float64) - g["slopes"]).max() <= \
            2 * np.spacing(np.abs(g["slopes"]).max().astype(np.float32))
    else:
        assert np.array_equal(v[:, cols], g["values"])
        assert np.array_equal(s[:, cols[cols < n - 1]], g["slopes"])
        assert np.array_equal(v.sum(axis=1), g["value_sums"])
    # table values interpolated by the fp32 kernel (float64 reference cell)
    t = g["points"].astype(np.float64)
    x = np.arctanh(np.clip(t, -1 + 1e-7, 1 - 1e-7)).astype(np.float32)
    tt = np.tanh(x.astype(np.float64))
    want_v, want_s = orc.lut_values_and_slopes(tt, *orc.build_table(degree, n, kind)[:2])
    phi, slopes = ck.expand(_t(x).reshape(1, -1), table, with_slopes=True)
    k = table.n_features
    scale = max(1.0, float(np.abs(want_v).max()))
    assert np.abs(phi.reshape(-1, k).cpu().numpy() - want_v).max() <= 4e-6 * scale


def _kind_layer(g, functional: bool):
    kind, degree, exact = ck.BasisKind(str(g["kind"])), int(g["degree"]), bool(g["exact"])
    i, o = g["x"].shape[1], g["dy"].shape[1]
    jac = bool(g["jacobian"])
    path = ck.BasisPath.EXACT_RECURRENCE if exact else ck.BasisPath.LUT_INTERP
    if functional:
        table = None if exact else ck.lut_build(kind, degree, int(g["lut_size"]), device=_dev())
        k = ck.feature_count(kind, degree)
        c = ck.reorder_to_doj(ck.CoeffTensor(i, o, k - 1, ck.Layout.JOD, _t(g["c_jod"])))
        bias = _t(g["bias"]) if "bias" in g else None
        mode = ck.KernelMode(path, include_tanh_jacobian=jac)
        y = ck.fused_forward(_t(g["x"]), c, table, None, mode, bias, kind=kind)
        cg, dx = ck.backward_fused(_t(g["x"]), c, _t(g["dy"]), table, None, mode, kind=kind)
        return y.cpu().numpy(), cg.data.cpu().numpy(), dx.cpu().numpy(), None
    layer = ck.ChebyKANLayer(i, o, degree, bias="bias" in g, lut_size=max(int(g["lut_size"]), 2),
                             include_tanh_jacobian=jac, kind=kind, basis_path=path).to(_dev())
    layer.load_jod(g["c_jod"])
    if "bias" in g:
        with torch.no_grad():
            layer.bias.copy_(_t(g["bias"]))
    x = _t(g["x"]).requires_grad_(True)
    y = layer(x)
    y.backward(_t(g["dy"]))
    db = layer.bias.grad.cpu().numpy() if "bias" in g else None
    return y.detach().cpu().numpy(), layer.coeff_doj.grad.cpu().numpy(), x.grad.cpu().numpy(), db


@pytest.mark.parametrize("functional", [True, False], ids=["functional", "module"])
@pytest.mark.parametrize("path", golden_kind_cases(), ids=lambda p: p.stem)
def test_kind_layers_match_reference_golden(path, functional):
    g = np.load(path)
    y, dc, dx, db = _kind_layer(g, functional)
    errs = {"y": orc.normwise_err(y, g["y"]), "dc": orc.normwise_err(dc, g["dc_doj"]),
            "dx": orc.normwise_err(dx, g["dx"])}
    if db is not None:
        errs["db"] = orc.normwise_err(db, g["db"])
    print(path.stem, {k: f"{v:.2e}" for k, v in errs.items()})
    for k, e in errs.items():
        assert e <= TOL, (k, e)


@pytest.mark.parametrize("path", [p for p in golden_kind_cases() if "exact_chebyshev" in p.stem],
                         ids=lambda p: p.stem)
def test_reference_kernels_trig_match_reference(path):
    # reference_forward / reference_backward with trig=True (kernels.py:450-510)
    g = np.load(path)
    i, o = g["x"].shape[1], g["dy"].shape[1]
    degree = int(g["degree"])
    c = ck.CoeffTensor(i, o, degree, ck.Layout.JOD, _t(g["c_jod"]))
    y = ck.reference_forward(_t(g["x"]), c, degree, trig=True).cpu().numpy()
    assert orc.normwise_err(y, g["y_ref_trig"]) <= TOL
    cg, dx = ck.reference_backward(_t(g["x"]), c, _t(g["dy"]), trig=True,
                                   include_tanh_jacobian=bool(g["jacobian"]))
    assert cg.layout is ck.Layout.JOD
    assert orc.normwise_err(cg.data.cpu().numpy(), g["dc_ref_trig_jod"]) <= TOL
    assert orc.normwise_err(dx.cpu().numpy(), g["dx_ref_trig"]) <= TOL


@pytest.mark.parametrize("kind", ["chebyshev", "legendre", "hermite", "fourier"])
@pytest.mark.parametrize("degree", [0, 1, 3, 8, 13])
def test_exact_expand_matches_basis_and_derivative_rows(kind, degree):
    rng = np.random.default_rng(degree)
    x = rng.uniform(-2.5, 2.5, 4000).astype(np.float32)
    basis = ck.exact_basis(ck.BasisKind(kind), degree, device=_dev())
    phi, dphi = ck.expand(_t(x).reshape(1, -1), basis, with_slopes=True)
    t = np.tanh(x.astype(np.float64))
    want_v = orc.basis_rows(kind, degree, t).T
    want_d = orc.derivative_rows(kind, degree, t).T
    k = want_v.shape[1]
    # float32 tanh (1-2 ulp) amplified by |B_k'| and the recurrence round-off
    assert orc.normwise_err(phi.reshape(-1, k).cpu().numpy(), want_v) <= 1e-5
    assert orc.normwise_err(dphi.reshape(-1, k).cpu().numpy(), want_d) <= 1e-5


@pytest.mark.parametrize("kind", ["legendre", "hermite", "fourier"])
def test_kind_random_shapes_vs_oracle(kind):
    # larger shapes than the golden files, through the tensor-core path
    b, i, o, d, n = 1024, 384, 320, 4, 4096
    k = orc.feature_count(kind, d)
    rng = np.random.default_rng(5)
    s = 1.0 / np.sqrt(i * k)
    x = rng.uniform(-1.5, 1.5, (b, i)).astype(np.float32)
    c_doj = rng.uniform(-s, s, (k, o, i)).astype(np.float32)
    dy = rng.standard_normal((b, o)).astype(np.float32)
    for exact in (False, True):
        if exact:
            wy = orc.exact_layer_forward(x, c_doj, kind, threads=8)
            wdc, wdx, _ = orc.exact_layer_backward(x, c_doj, dy, kind, threads=8)
            table, mode = None, ck.EXACT_MODE
        else:
            vals, slopes, _ = orc.build_table(d, n, kind)
            wy = orc.layer_forward(x, c_doj, vals, threads=8)
            wdc, wdx, _ = orc.layer_backward(x, c_doj, dy, vals, slopes, threads=8)
            table, mode = ck.lut_build(ck.BasisKind(kind), d, n, device=_dev()), ck.LUT_MODE
        c = ck.CoeffTensor(i, o, k - 1, ck.Layout.DOJ, _t(c_doj))
        y = ck.fused_forward(_t(x), c, table, None, mode, kind=ck.BasisKind(kind)).cpu().numpy()
        cg, dx = ck.backward_fused(_t(x), c, _t(dy), table, None, mode, kind=ck.BasisKind(kind))
        e = (orc.normwise_err(y, wy), orc.normwise_err(cg.data.cpu().numpy(), wdc),
             orc.normwise_err(dx.cpu().numpy(), wdx))
        print(kind, "exact" if exact else "lut", [f"{v:.2e}" for v in e])
        assert max(e) <= TOL, e


def test_exact_mode_error_paths():
    c = ck.CoeffTensor(3, 2, 2, ck.Layout.DOJ, torch.ones(18, device=_dev()))
    with pytest.raises(ValueError, match="exact mode without a LUT requires an explicit basis kind"):
        ck.fused_forward(torch.zeros(1, 3, device=_dev()), c, None, None, ck.EXACT_MODE)
    with pytest.raises(ValueError, match="Fourier feature count must be odd"):
        ck.fused_forward(torch.zeros(1, 3, device=_dev()), c.__class__(3, 2, 1, ck.Layout.DOJ,
                         torch.ones(12, device=_dev())), None, None, ck.EXACT_MODE, kind=ck.BasisKind.FOURIER)
    cj = ck.CoeffTensor(3, 2, 2, ck.Layout.JOD, torch.ones(18, device=_dev()))
    with pytest.raises(ValueError, match="trig path applies to the Chebyshev basis only"):
        ck.reference_forward(torch.zeros(1, 3, device=_dev()), cj, 2, trig=True, kind=ck.BasisKind.HERMITE)


@pytest.mark.parametrize("o,d,kind,exact", [(1, 5, "chebyshev", False), (2, 7, "legendre", False),
                                            (3, 3, "fourier", False), (4, 6, "chebyshev", True),
                                            (8, 3, "hermite", False), (1, 20, "chebyshev", False),
                                            (5, 2, "hermite", True)])
def test_skinny_output_layers_vs_oracle(o, d, kind, exact):
    # d_out <= 8 runs on the CUDA-core skinny kernels (no tensor-core tiles)
    b, i, n = 3000, 515, 4096
    k = orc.feature_count(kind, d)
    rng = np.random.default_rng(o * 100 + d)
    s = 1.0 / np.sqrt(i * k)
    x = rng.uniform(-2, 2, (b, i)).astype(np.float32)
    c_doj = rng.uniform(-s, s, (k, o, i)).astype(np.float32)
    dy = rng.standard_normal((b, o)).astype(np.float32)
    bias = rng.standard_normal(o).astype(np.float32) * 0.1
    if exact:
        wy = orc.exact_layer_forward(x, c_doj, kind, bias.astype(np.float64), threads=8)
        wdc, wdx, wdb = orc.exact_layer_backward(x, c_doj, dy, kind, threads=8)
        table, mode = None, ck.EXACT_MODE
    else:
        vals, slopes, _ = orc.build_table(d, n, kind)
        wy = orc.layer_forward(x, c_doj, vals, bias.astype(np.float64), threads=8)
        wdc, wdx, wdb = orc.layer_backward(x, c_doj, dy, vals, slopes, threads=8)
        table, mode = ck.lut_build(ck.BasisKind(kind), d, n, device=_dev()), ck.LUT_MODE
    c = ck.CoeffTensor(i, o, k - 1, ck.Layout.DOJ, _t(c_doj))
    y = ck.fused_forward(_t(x), c, table, None, mode, _t(bias), kind=ck.BasisKind(kind)).cpu().numpy()
    outs = []
    for _ in range(2):
        cg, dx = ck.backward_fused(_t(x), c, _t(dy), table, None, mode, kind=ck.BasisKind(kind))
        outs.append((cg.data.clone(), dx.clone()))
    assert all(torch.equal(a, bb) for a, bb in zip(outs[0], outs[1]))  # deterministic two-stage merge
    e = (orc.normwise_err(y, wy), orc.normwise_err(outs[0][0].cpu().numpy(), wdc),
         orc.normwise_err(outs[0][1].cpu().numpy(), wdx))
    print((o, d, kind, exact), [f"{v:.2e}" for v in e])
    assert max(e) <= TOL, e
    # bias gradient through the module path
    layer = ck.ChebyKANLayer(i, o, d, kind=ck.BasisKind(kind), lut_size=n,
                             basis_path=ck.BasisPath.EXACT_RECURRENCE if exact else ck.BasisPath.LUT_INTERP).to(_dev())
    with torch.no_grad():
        layer.coeff_doj.copy_(_t(c_doj))
    layer(_t(x)).backward(_t(dy))
    assert orc.normwise_err(layer.bias.grad.cpu().numpy(), wdb) <= 1e-6


@pytest.mark.parametrize("o", [40, 3])
def test_empty_batch(o):
    # batch 0: y is (0, O), dC and db are zeros, dX is (0, I) -- both the
    # tensor-core path and the skinny path
    table = ck.lut_build(ck.BasisKind.CHEBYSHEV, 4, 1024, device=_dev())
    c = ck.CoeffTensor(24, o, 4, ck.Layout.DOJ, torch.randn(5, o, 24, device=_dev()))
    x = torch.zeros(0, 24, device=_dev())
    y = ck.fused_forward(x, c, table)
    assert tuple(y.shape) == (0, o)
    cg, dx = ck.backward_fused(x, c, torch.zeros(0, o, device=_dev()), table)
    assert tuple(dx.shape) == (0, 24) and torch.count_nonzero(cg.data) == 0
    layer = ck.ChebyKANLayer(24, o, 4, lut_size=1024).to(_dev())
    xx = torch.zeros(0, 24, device=_dev(), requires_grad=True)
    layer(xx).sum().backward()
    assert torch.count_nonzero(layer.coeff_doj.grad) == 0 and torch.count_nonzero(layer.bias.grad) == 0


def test_multi_chunk_batch_vs_oracle():
    # 70000 rows = 3 internal 32768-row chunks (ragged last): dC accumulates
    # across chunks in ascending order, the basis cache holds one slot per
    # chunk, db sums per-chunk row-block partials
    b, i, o, d, n = 70000, 64, 48, 3, 2048
    x, c_jod, dy = orc.bench_inputs(b, i, o, d, seed=11)
    vals, slopes, _ = orc.build_table(d, n)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    want_y = orc.layer_forward(x, c_doj, vals, threads=8)
    want_dc, want_dx, want_db = orc.layer_backward(x, c_doj, dy, vals, slopes, threads=8)
    layer = ck.ChebyKANLayer(i, o, d, lut_size=n).to(_dev())
    layer.load_jod(c_jod)
    xt = _t(x).requires_grad_(True)
    y = layer(xt)
    y.backward(_t(dy))
    errs = (orc.normwise_err(y.detach().cpu().numpy(), want_y),
            orc.normwise_err(layer.coeff_doj.grad.cpu().numpy(), want_dc),
            orc.normwise_err(xt.grad.cpu().numpy(), want_dx),
            orc.normwise_err(layer.bias.grad.cpu().numpy(), want_db))
    print("multi-chunk", [f"{e:.2e}" for e in errs])
    assert max(errs) <= TOL, errs


_GEN_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2511_14852_b200 as ck
from paper_2511_14852_b200 import _lib
from oracle import chebykan_oracle as orc
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
worst = 0.0
for (b, i, o, d, n, kind) in {cases!r}:
    k = orc.feature_count(kind, d)
    rng = np.random.default_rng(b + i + o + d)
    s = 1.0 / np.sqrt(i * k)
    x = rng.uniform(-1.5, 1.5, (b, i)).astype(np.float32)
    c_doj = rng.uniform(-s, s, (k, o, i)).astype(np.float32)
    bias = rng.standard_normal(o).astype(np.float32)
    if n == 0:
        want = orc.exact_layer_forward(x, c_doj, kind, bias=bias, threads=8)
        table, mode = None, ck.EXACT_MODE
    else:
        vals, _, _ = orc.build_table(d, n, kind)
        want = orc.layer_forward(x, c_doj, vals, bias=bias, threads=8)
        table, mode = ck.lut_build(ck.BasisKind(kind), d, n, device=dev), ck.LUT_MODE
    c = ck.CoeffTensor(i, o, k - 1, ck.Layout.DOJ, t(c_doj))
    _lib.timing_collect()
    _lib.timing_enable(True)
    y = ck.fused_forward(t(x), c, table, mode=mode, bias=t(bias), kind=ck.BasisKind(kind)).cpu().numpy()
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    assert kt.get("expand", (0, 0))[1] == 0, ("planes were materialised", kt)
    y2 = ck.fused_forward(t(x), c, table, mode=mode, bias=t(bias), kind=ck.BasisKind(kind)).cpu().numpy()
    assert np.array_equal(y, y2), "generated forward not bitwise reproducible"
    e = orc.normwise_err(y, want)
    print((b, i, o, d, n, kind), f"{{e:.2e}}")
    worst = max(worst, e)
print("WORST", worst)
"""


def test_generated_forward_vs_oracle():
    """The forward with the basis generated in shared memory (ck_gemm_gen.cu)
    on every degree class and basis family, ragged inputs / outputs, two N
    tiles, LUT and exact mode -- in a subprocess with CK_GEN=all (the default
    rule only picks it for d >= 4, d*I >= 1536)."""
    import os
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    cases = [(300, 257, 130, 3, 512, "chebyshev"), (2048, 512, 256, 5, 1024, "chebyshev"),
             (96, 40, 300, 16, 32768, "chebyshev"), (1000, 100, 60, 1, 4096, "chebyshev"),
             (5000, 129, 256, 8, 32768, "chebyshev"), (700, 64, 200, 2, 2048, "chebyshev"),
             (513, 130, 96, 11, 32768, "chebyshev"), (600, 96, 128, 6, 0, "chebyshev"),
             (700, 200, 160, 5, 4096, "legendre"), (400, 96, 64, 7, 0, "legendre"),
             (700, 200, 160, 4, 4096, "hermite"), (400, 96, 64, 3, 0, "hermite"),
             (700, 200, 160, 3, 4096, "fourier"), (400, 96, 64, 8, 0, "fourier")]
    script = _GEN_SCRIPT.format(root=str(root), tests=str(root / "tests"), cases=cases)
    env = dict(os.environ, CK_GEN="all", CK_GEN_MAX_O="512")
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0
    worst = float(out.stdout.strip().splitlines()[-1].split()[1])
    assert worst <= TOL, worst
