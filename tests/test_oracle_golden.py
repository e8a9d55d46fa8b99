"""Pin the CPU oracle to golden vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py, which runs the
reference's fused_forward / backward_fused / lut_build.  The oracle must
reproduce them to float64 round-off (BLAS summation order is the only
allowed difference).
"""
import numpy as np
import pytest

from conftest import GOLDEN, golden_kind_cases, golden_kind_lut_cases, golden_layer_cases, golden_lut_cases
from oracle import chebykan_oracle as orc


def test_lut_known_answer_d2_n3():
    g = np.load(GOLDEN / "lut_kat_d2_n3.npz")
    values, slopes, step = orc.build_table(2, 3)
    assert step == 1.0 == float(g["step"])
    assert np.array_equal(values, g["values"])
    assert np.array_equal(slopes, g["slopes"])
    # test_lut.py:29-33 literal values
    assert np.array_equal(values, [[1, 1, 1], [-1, 0, 1], [1, -1, 1]])
    assert np.array_equal(slopes, [[0, 0], [1, 1], [-2, 2]])
    # test_lut.py:81-85: lerp of T_2 at 0.5 on the coarse table is 0
    np.testing.assert_allclose(orc.lut_values(np.array([0.5]), values)[0], [1.0, 0.5, 0.0], atol=1e-15)
    # test_lut.py:96-99: left-cell slope example
    _, s = orc.lut_values_and_slopes(np.array([-0.4]), values, slopes)
    assert s[0, 2] == -2.0


@pytest.mark.parametrize("path", golden_lut_cases(), ids=lambda p: p.stem)
def test_lut_tables_and_interp_match_reference(path):
    g = np.load(path)
    degree = int(path.stem.split("_")[1][1:])
    n = int(path.stem.split("_")[2][1:])
    values, slopes, step = orc.build_table(degree, n)
    assert step == float(g["step"])
    cols = g["cols"]
    assert np.array_equal(values[:, cols], g["values"])
    assert np.array_equal(slopes[:, cols[cols < n - 1]], g["slopes"])
    assert np.array_equal(values.sum(axis=1), g["value_sums"])
    assert np.array_equal(slopes.astype(np.float64).sum(axis=1), g["slope_sums"])
    pts = g["points"].astype(np.float64)
    v, s = orc.lut_values_and_slopes(pts, values, slopes)
    assert np.array_equal(v, g["interp"])
    assert np.array_equal(s, g["interp_slopes"])
    assert np.array_equal(orc.interp_error_bound(degree, n), g["bound"])


@pytest.mark.parametrize("path", golden_layer_cases(), ids=lambda p: p.stem)
def test_layer_forward_backward_match_reference(path):
    g = np.load(path)
    degree, n = int(g["degree"]), int(g["lut_size"])
    values, slopes, _ = orc.build_table(degree, n)
    c_doj = orc.jod_to_doj(g["c_jod"].astype(np.float64))
    bias = g["bias"].astype(np.float64) if "bias" in g else None
    x = g["x"].astype(np.float64)
    y = orc.layer_forward(x, c_doj, values, bias)
    dc, dx, db = orc.layer_backward(x, c_doj, g["dy"], values, slopes,
                                    include_tanh_jacobian=bool(g["jacobian"]))
    # Identical algorithm and tile order: expect bitwise equality; allow
    # 1e-13 normwise for BLAS kernel-selection differences.
    for got, want in ((y, g["y"]), (dc, g["dc_doj"]), (dx, g["dx"]), (db, g["db"])):
        assert got.shape == want.shape
        assert orc.normwise_err(got, want) <= 1e-13
    ye = orc.exact_forward(x, c_doj, bias)
    assert orc.normwise_err(ye, g["y_exact"]) <= 1e-13


def test_oracle_threads_do_not_change_results():
    g = np.load(GOLDEN / "layer_ragged_257x96_d8_n1024.npz")
    values, slopes, _ = orc.build_table(8, 1024)
    c_doj = orc.jod_to_doj(g["c_jod"].astype(np.float64))
    x = g["x"].astype(np.float64)
    y1 = orc.layer_forward(x, c_doj, values, threads=1)
    y4 = orc.layer_forward(x, c_doj, values, threads=4)
    assert np.array_equal(y1, y4)
    a = orc.layer_backward(x, c_doj, g["dy"], values, slopes, threads=1)
    b = orc.layer_backward(x, c_doj, g["dy"], values, slopes, threads=4)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_interp_error_vs_exact_within_bound():
    # lut.py:143-153 closed form bounds the measured error (test_lut.py:125-129).
    for degree, n in ((8, 1024), (8, 4096), (3, 512)):
        values, _, _ = orc.build_table(degree, n)
        t = np.linspace(-1.0, 1.0, 20001)
        err = np.abs(orc.lut_values(t, values).T - orc.chebyshev_rows(degree, t)).max(axis=1)
        assert (err <= orc.interp_error_bound(degree, n) * (1 + 1e-6) + 1e-12).all()


@pytest.mark.parametrize("path", golden_kind_lut_cases(), ids=lambda p: p.stem)
def test_kind_lut_tables_match_reference(path):
    # Legendre / Hermite / Fourier tables (lut.py:76-94 over basis.py:87-119)
    g = np.load(path)
    kind, degree, n = str(g["kind"]), int(g["degree"]), int(g["lut_size"])
    values, slopes, step = orc.build_table(degree, n, kind)
    assert step == float(g["step"])
    cols = g["cols"]
    assert np.array_equal(values[:, cols], g["values"])
    assert np.array_equal(slopes[:, cols[cols < n - 1]], g["slopes"])
    assert np.array_equal(values.sum(axis=1), g["value_sums"])
    v, s = orc.lut_values_and_slopes(g["points"].astype(np.float64), values, slopes)
    assert np.array_equal(v, g["interp"])
    assert np.array_equal(s, g["interp_slopes"])


@pytest.mark.parametrize("path", golden_kind_cases(), ids=lambda p: p.stem)
def test_kind_layers_match_reference(path):
    g = np.load(path)
    kind, degree, exact = str(g["kind"]), int(g["degree"]), bool(g["exact"])
    c_doj = orc.jod_to_doj(g["c_jod"].astype(np.float64))
    bias = g["bias"].astype(np.float64) if "bias" in g else None
    x = g["x"].astype(np.float64)
    jac = bool(g["jacobian"])
    if exact:
        y = orc.exact_layer_forward(x, c_doj, kind, bias)
        dc, dx, db = orc.exact_layer_backward(x, c_doj, g["dy"], kind, include_tanh_jacobian=jac)
    else:
        values, slopes, _ = orc.build_table(degree, int(g["lut_size"]), kind)
        y = orc.layer_forward(x, c_doj, values, bias)
        dc, dx, db = orc.layer_backward(x, c_doj, g["dy"], values, slopes, include_tanh_jacobian=jac)
    for got, want in ((y, g["y"]), (dc, g["dc_doj"]), (dx, g["dx"]), (db, g["db"])):
        assert got.shape == want.shape
        assert orc.normwise_err(got, want) <= 1e-13
    if "y_ref_trig" in g:
        yt = orc.exact_forward(x, c_doj)
        assert orc.normwise_err(yt + (0 if bias is None else 0), g["y_ref_trig"]) <= 1e-12


def test_reference_basis_known_answers():
    # test_basis.py:20-26, 70-77, 90-96 / kernels: closed forms
    assert np.array_equal(orc.basis_rows("legendre", 2, np.array([1.0]))[:, 0], [1.0, 1.0, 1.0])
    x = 0.37
    want = [1.0]
    for k in range(1, 4):
        want += [np.cos(k * np.pi * x), np.sin(k * np.pi * x)]
    np.testing.assert_allclose(orc.basis_rows("fourier", 3, np.array([x]))[:, 0], want, atol=1e-12)
    h = orc.basis_rows("hermite", 3, np.array([x]))[:, 0]
    np.testing.assert_allclose(h, [1, 2 * x, 4 * x * x - 2, 8 * x ** 3 - 12 * x], atol=1e-12)
    np.testing.assert_allclose(orc.derivative_rows("fourier", 1, np.array([0.0]))[:, 0], [0, 0, np.pi], atol=1e-15)
