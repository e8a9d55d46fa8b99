"""The reference's own kernel tests (pkg/tests/test_kernels.py), ported to the
B200 path: random-instance sweeps in both basis paths and all families,
finite-difference gradient checks, the pseudocode-literal (no-Jacobian)
relation, schedule independence and the closed-form merge counters."""
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
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=_dev())


def random_instance(rng, kind="chebyshev", max_dim=64, max_degree=24, x_range=2.0):
    """test_kernels.py:31-43, float32-representable, any family."""
    batch = int(rng.integers(1, 17))
    d_in = int(rng.integers(1, max_dim + 1))
    d_out = int(rng.integers(1, max_dim + 1))
    degree = int(rng.integers(0, max_degree + 1))
    k = orc.feature_count(kind, degree)
    x = rng.uniform(-x_range, x_range, size=(batch, d_in)).astype(np.float32)
    s = 1.0 / np.sqrt(d_in * k)
    c_doj = rng.uniform(-s, s, size=(k, d_out, d_in)).astype(np.float32)
    dy = rng.standard_normal((batch, d_out)).astype(np.float32)
    return x, c_doj, dy, degree


@pytest.mark.parametrize("kind", ["chebyshev", "legendre", "hermite", "fourier"])
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "lut"])
def test_random_instance_sweep(kind, exact):
    # test_fused_exact_equals_reference_sweep (test_kernels.py:104-111) in both paths
    rng = np.random.default_rng(13 + len(kind))
    for _ in range(12):
        x, c_doj, dy, degree = random_instance(rng, kind, max_dim=48,
                                               max_degree=12 if kind == "fourier" else 24)
        k = c_doj.shape[0]
        if exact:
            wy = orc.exact_layer_forward(x, c_doj, kind)
            wdc, wdx, _ = orc.exact_layer_backward(x, c_doj, dy, kind)
            table, mode = None, ck.EXACT_MODE
        else:
            vals, slopes, _ = orc.build_table(degree, 4096, kind)
            wy = orc.layer_forward(x, c_doj, vals)
            wdc, wdx, _ = orc.layer_backward(x, c_doj, dy, vals, slopes)
            table, mode = ck.lut_build(ck.BasisKind(kind), degree, 4096, device=_dev()), ck.LUT_MODE
        c = ck.CoeffTensor(x.shape[1], dy.shape[1], k - 1, ck.Layout.DOJ, _t(c_doj))
        y = ck.fused_forward(_t(x), c, table, None, mode, kind=ck.BasisKind(kind)).cpu().numpy()
        cg, dx = ck.backward_fused(_t(x), c, _t(dy), table, None, mode, kind=ck.BasisKind(kind))
        errs = [orc.normwise_err(y, wy), orc.normwise_err(cg.data.cpu().numpy(), wdc)]
        if degree > 0:
            errs.append(orc.normwise_err(dx.cpu().numpy(), wdx))
        else:
            assert torch.count_nonzero(dx) == 0
        assert max(errs) <= TOL, (x.shape, dy.shape, degree, errs)


def test_lut_coeff_grad_matches_forward_differences():
    # test_kernels.py:230-256: y is linear in C, so central differences of the
    # (GPU) forward reproduce the (GPU) coefficient gradient
    rng = np.random.default_rng(18)
    batch, d_in, d_out, degree = 2, 4, 3, 5
    x = rng.uniform(-1.5, 1.5, (batch, d_in)).astype(np.float32)
    c_doj = rng.uniform(-0.5, 0.5, (degree + 1, d_out, d_in)).astype(np.float32)
    dy = rng.standard_normal((batch, d_out)).astype(np.float32)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, degree, 32768, device=_dev())
    c = ck.CoeffTensor(d_in, d_out, degree, ck.Layout.DOJ, _t(c_doj))
    cg, _ = ck.backward_fused(_t(x), c, _t(dy), lut)
    cg = cg.data.cpu().numpy().reshape(-1)
    h = 0.25
    flat = c_doj.reshape(-1)
    for i in range(flat.size):
        cp, cm = flat.copy(), flat.copy()
        cp[i] += h
        cm[i] -= h
        f = [float((ck.fused_forward(_t(x), ck.CoeffTensor(d_in, d_out, degree, ck.Layout.DOJ,
                                                           _t(v.reshape(c_doj.shape))), lut).cpu().numpy()
                    * dy).sum()) for v in (cp, cm)]
        fd = (f[0] - f[1]) / (2 * h)
        assert abs(cg[i] - fd) / max(abs(fd), 1e-3) <= 1e-3


def test_exact_x_grad_matches_finite_differences():
    # test_kernels.py:211-227 (exact mode): FD of the float64 reference forward
    rng = np.random.default_rng(17)
    for _ in range(5):
        x, c_doj, dy, degree = random_instance(rng, max_dim=10, max_degree=8, x_range=1.5)
        c = ck.CoeffTensor(x.shape[1], dy.shape[1], degree, ck.Layout.DOJ, _t(c_doj))
        _, xg = ck.backward_fused(_t(x), c, _t(dy), None, None, ck.EXACT_MODE, kind=ck.BasisKind.CHEBYSHEV)
        xg = xg.cpu().numpy()
        h = 1e-5
        for _ in range(4):
            b = int(rng.integers(0, x.shape[0]))
            j = int(rng.integers(0, x.shape[1]))
            xp, xm = x.astype(np.float64), x.astype(np.float64)
            xp[b, j] += h
            xm[b, j] -= h
            fd = ((orc.exact_layer_forward(xp, c_doj) * dy).sum() - (orc.exact_layer_forward(xm, c_doj) * dy).sum()) / (
                2 * h)
            scale = max(np.abs(xg).max(), 1e-3)
            assert abs(xg[b, j] - fd) <= 1e-3 * scale


def test_backward_without_jacobian_matches_pseudocode_literal():
    # test_kernels.py:178-189: chain-rule dX = literal dX * (1 - tanh^2)
    rng = np.random.default_rng(15)
    x, c_doj, dy, degree = random_instance(rng, max_dim=12, max_degree=6)
    degree = max(degree, 1)
    c_doj = rng.uniform(-0.3, 0.3, (degree + 1, dy.shape[1], x.shape[1])).astype(np.float32)
    c = ck.CoeffTensor(x.shape[1], dy.shape[1], degree, ck.Layout.DOJ, _t(c_doj))
    for mode_j, mode_p in ((ck.EXACT_MODE, ck.KernelMode(ck.BasisPath.EXACT_RECURRENCE, False)),):
        _, plain = ck.backward_fused(_t(x), c, _t(dy), None, None, mode_p, kind=ck.BasisKind.CHEBYSHEV)
        _, chain = ck.backward_fused(_t(x), c, _t(dy), None, None, mode_j, kind=ck.BasisKind.CHEBYSHEV)
        t = np.tanh(x.astype(np.float64))
        np.testing.assert_allclose(chain.cpu().numpy(), plain.cpu().numpy() * (1 - t * t), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("kind,exact", [("chebyshev", False), ("legendre", True), ("fourier", False)])
def test_forward_partial_and_combine(kind, exact):
    # kernels.py:263-348 stage by stage: every slot vs the float64 tile sums,
    # one writer per real slot, padding lanes untouched, combine == fused_forward
    rng = np.random.default_rng(31)
    for tile_in, tile_out in ((4, 8), (16, 32), (64, 32), (64, 40)):
        x, c_doj, dy, degree = random_instance(rng, kind, max_dim=70, max_degree=8)
        b, i = x.shape
        o, k = c_doj.shape[1], c_doj.shape[0]
        sched = ck.TileSchedule.for_dims(i, o, tile_in, tile_out, lane_y=tile_out)
        if exact:
            planes = orc.basis_rows(kind, degree, np.tanh(x.astype(np.float64)))
            table, mode = None, ck.EXACT_MODE
        else:
            vals, _, _ = orc.build_table(degree, 4096, kind)
            planes = orc.lut_values(np.tanh(x.astype(np.float64)), vals).transpose(2, 0, 1)
            table, mode = ck.lut_build(ck.BasisKind(kind), degree, 4096, device=_dev()), ck.LUT_MODE
        c = ck.CoeffTensor(i, o, k - 1, ck.Layout.DOJ, _t(c_doj))
        buf = ck.PartialBuffer.allocate(sched, b, instrument=True, device=_dev())
        counters = ck.KernelCounters()
        ck.forward_partial(_t(x), c, table, sched, mode, buf, counters=counters, kind=ck.BasisKind(kind))
        got = buf.data.cpu().numpy()
        want = np.zeros_like(got, dtype=np.float64)
        for to in range(sched.g_y):
            os_ = slice(to * tile_out, min(o, (to + 1) * tile_out))
            for ti in range(sched.g_x):
                js = slice(ti * tile_in, min(i, (ti + 1) * tile_in))
                prod = np.einsum("kbj,koj->bo", planes[:, :, js], c_doj[:, os_, js].astype(np.float64))
                want[to, ti, :, : os_.stop - os_.start] = prod
        assert orc.normwise_err(got, want) <= 1e-5
        counts = buf.write_counts.cpu().numpy()
        assert set(np.unique(counts)) <= {0, 1}
        assert int(counts.sum()) == b * o * sched.g_x  # padding lanes excluded
        assert counters.partial_writes == b * o * sched.g_x
        bias = rng.standard_normal(o).astype(np.float32)
        y = ck.combine(buf, sched, _t(bias), counters=counters).cpu().numpy()
        yf = ck.fused_forward(_t(x), c, table, sched, mode, _t(bias), kind=ck.BasisKind(kind)).cpu().numpy()
        assert orc.normwise_err(y, yf) <= TOL
        assert counters.combine_stores == b * o


def test_point_evaluation_known_answers():
    # test_basis.py:20-110 and test_lut.py:29-99 through ck_basis_eval (float32)
    K = ck.BasisKind
    assert np.array_equal(ck.eval_basis(K.CHEBYSHEV, 2, 1.0), [1.0, 1.0, 1.0])
    assert np.array_equal(ck.eval_basis(K.LEGENDRE, 2, 1.0), [1.0, 1.0, 1.0])
    np.testing.assert_allclose(ck.eval_basis(K.CHEBYSHEV, 3, 0.5), [1.0, 0.5, -0.5, -1.0], atol=1e-6)
    np.testing.assert_allclose(ck.eval_basis_trig(3, 0.5), [1.0, 0.5, -0.5, -1.0], atol=1e-6)
    np.testing.assert_allclose(ck.eval_basis_trig(4, -1.0), [1, -1, 1, -1, 1], atol=1e-6)
    x = 0.37
    want = [1.0]
    for k in range(1, 4):
        want += [np.cos(k * np.pi * x), np.sin(k * np.pi * x)]
    np.testing.assert_allclose(ck.eval_basis(K.FOURIER, 3, x), want, atol=1e-6)
    np.testing.assert_allclose(ck.eval_basis(K.HERMITE, 3, x), [1, 2 * x, 4 * x * x - 2, 8 * x ** 3 - 12 * x],
                               atol=1e-5)
    np.testing.assert_allclose(ck.eval_basis_derivative(K.FOURIER, 1, 0.0), [0.0, 0.0, np.pi], atol=1e-6)
    for kind in ("chebyshev", "legendre", "hermite", "fourier"):
        xs = np.linspace(-1, 1, 2001).astype(np.float32).astype(np.float64)  # the kernels' float32 points
        for deg in (0, 5, 12):
            tol = 1e-7 * (deg + 1) ** 2  # float32 recurrence round-off grows ~k^2 ulp
            got = ck.basis_rows(K(kind), deg, xs)
            want = orc.basis_rows(kind, deg, xs)
            assert got.shape == want.shape
            assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max())
            gd, wd = ck.derivative_rows(K(kind), deg, xs), orc.derivative_rows(kind, deg, xs)
            assert np.abs(gd - wd).max() <= tol * max(1.0, np.abs(wd).max())
    with pytest.raises(ValueError, match="trig evaluation requires"):
        ck.trig_rows(3, np.array([1.5]))
    with pytest.raises(ValueError, match="finite inputs"):
        ck.basis_rows(K.CHEBYSHEV, 3, np.array([np.nan]))
    with pytest.raises(ValueError, match="takes a scalar"):
        ck.eval_basis(K.CHEBYSHEV, 3, np.zeros(2))
    # coarse table KATs (test_lut.py:81-99): lerp of T_2 at 0.5 is 0; cell-0 slope of T_2 is -2
    t = ck.lut_build(K.CHEBYSHEV, 2, 3, device=_dev())
    np.testing.assert_allclose(ck.lut_interp(t, 0.5), [1.0, 0.5, 0.0], atol=1e-7)
    _, s = ck.lut_interp_with_slope(t, -0.4)
    assert s[2] == -2.0
    # grid points reproduce stored columns (snap), and batch interp == oracle
    t = ck.lut_build(K.LEGENDRE, 6, 1025, device=_dev())
    grid = t.grid()
    v = ck.interp_rows(t, grid)
    assert np.array_equal(v, t.values.T.astype(np.float32).astype(np.float64))
    pts = np.random.default_rng(3).uniform(-1.2, 1.2, 5000)
    vals, slopes = ck.interp_rows_with_slope(t, pts.astype(np.float32))
    wv, ws = orc.lut_values_and_slopes(pts.astype(np.float32).astype(np.float64), *orc.build_table(6, 1025, "legendre")[:2])
    assert np.abs(vals - wv).max() <= 2e-6
    assert np.array_equal(slopes, ws)


@pytest.mark.parametrize("o", [1, 96])
def test_saturated_inputs_use_the_last_cell(o):
    # tanh(+-inf) = +-1 and |x| >= 10 saturate; the reference clamps the cell to
    # N-2 (lut.py:101-103): the LUT-mode slopes (no Jacobian, so they reach dX
    # unscaled) and values at the ends of the table, on the tensor-core path
    # (o = 96) and the skinny path (o = 1)
    rng = np.random.default_rng(31)
    b, i, d, n = 257, 40, 5, 1024
    x = rng.uniform(-1.5, 1.5, (b, i)).astype(np.float32)
    x[::7, 0] = np.inf
    x[1::7, 1] = -np.inf
    x[2::7, 2] = 1e30
    x[3::7, 3] = -1e30
    x[4::7, 4] = 20.0
    c_doj = rng.uniform(-0.3, 0.3, (d + 1, o, i)).astype(np.float32)
    dy = rng.standard_normal((b, o)).astype(np.float32)
    vals, slopes, _ = orc.build_table(d, n)
    want_y = orc.layer_forward(x, c_doj, vals)
    want_dc, want_dx, _ = orc.layer_backward(x, c_doj, dy, vals, slopes, include_tanh_jacobian=False)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, d, n, device=_dev())
    c = ck.CoeffTensor(i, o, d, ck.Layout.DOJ, _t(c_doj))
    mode = ck.KernelMode(ck.BasisPath.LUT_INTERP, False)
    y = ck.fused_forward(_t(x), c, lut, None, mode).cpu().numpy()
    cg, dx = ck.backward_fused(_t(x), c, _t(dy), lut, None, mode)
    assert orc.normwise_err(y, want_y) <= 1e-4
    assert orc.normwise_err(cg.data.cpu().numpy(), want_dc) <= 1e-4
    assert orc.normwise_err(dx.cpu().numpy(), want_dx) <= 1e-4
