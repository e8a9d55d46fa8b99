"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is not present on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case calls the reference's own public API -- ``lut_build``
(lut.py:76), ``interp_rows_with_slope`` (lut.py:118), ``fused_forward``
(kernels.py:351), ``backward_fused`` (kernels.py:374), ``reference_forward``
(kernels.py:450) and ``Layer.backward``'s bias rule (model.py:147) -- on
float32-representable inputs, and stores inputs plus float64 outputs in
``tests/golden/*.npz``.  The oracle (oracle/chebykan_oracle.py) and the CUDA
path are both checked against these files.
"""
from __future__ import annotations

import pathlib

import numpy as np

from polykan.basis import BasisKind, feature_count
from polykan.kernels import (
    BasisPath,
    KernelMode,
    LUT_MODE,
    TileSchedule,
    backward_fused,
    fused_forward,
    reference_forward,
)
from polykan.kernels import EXACT_MODE, reference_backward
from polykan.lut import interp_rows_with_slope, lut_build, lut_max_error_bound
from polykan.tensor import CoeffTensor, Layout, reorder_to_doj

HERE = pathlib.Path(__file__).resolve().parent
CHEB = BasisKind.CHEBYSHEV

# (name, batch, d_in, d_out, degree, lut_size, seed, x_range, with_bias, jacobian)
LAYER_CASES = [
    ("tiny_d8_n32768", 4, 40, 16, 8, 32768, 11, 2.0, False, True),
    ("c0_b1024_64x64_d4_n4096", 1024, 64, 64, 4, 4096, 0, 1.5, True, True),
    ("ragged_257x96_d8_n1024", 33, 257, 96, 8, 1024, 5, 2.0, True, True),
    ("ragged_130x257_d3_n512", 65, 130, 257, 3, 512, 6, 2.0, True, True),
    ("degree0_n1024", 7, 20, 9, 0, 1024, 7, 2.0, True, True),
    ("degree1_n2048", 9, 17, 5, 1, 2048, 8, 2.0, True, True),
    ("head_o1_64_d5_n1024", 48, 64, 1, 5, 1024, 9, 2.0, True, True),
    ("single_1x1_d5_n1024", 1, 1, 1, 5, 1024, 10, 2.0, True, True),
    ("speech_257x24_d15_n16384", 24, 257, 24, 15, 16384, 12, 3.0, True, True),
    ("nojacobian_24x12_d6_n4096", 6, 24, 12, 6, 4096, 13, 2.0, False, False),
    ("wide_320x96_d8_n4096", 32, 320, 96, 8, 4096, 14, 1.5, True, True),
]


# Other basis families (LUT mode) and the exact-evaluation path (all kinds):
# (name, kind, exact, batch, d_in, d_out, degree, lut_size, seed, x_range, with_bias, jacobian)
KIND_CASES = [
    ("legendre_d6_n4096", "legendre", 0, 40, 72, 48, 6, 4096, 31, 2.0, True, True),
    ("hermite_d5_n2048", "hermite", 0, 33, 65, 40, 5, 2048, 32, 2.0, True, True),
    ("fourier_d4_n8192", "fourier", 0, 24, 48, 33, 4, 8192, 33, 2.0, True, True),
    ("fourier_d8_n32768", "fourier", 0, 20, 40, 24, 8, 32768, 34, 1.5, False, True),
    ("legendre_d20_n16384", "legendre", 0, 12, 30, 20, 20, 16384, 35, 2.0, True, True),
    ("hermite_d3_nojac_n1024", "hermite", 0, 9, 17, 5, 3, 1024, 36, 2.0, False, False),
    ("exact_chebyshev_d8", "chebyshev", 1, 32, 96, 40, 8, 0, 41, 2.0, True, True),
    ("exact_legendre_d5", "legendre", 1, 24, 64, 33, 5, 0, 42, 2.0, True, True),
    ("exact_hermite_d4", "hermite", 1, 17, 40, 24, 4, 0, 43, 2.0, False, True),
    ("exact_fourier_d3", "fourier", 1, 20, 33, 16, 3, 0, 44, 2.0, True, True),
    ("exact_chebyshev_d24", "chebyshev", 1, 10, 24, 12, 24, 0, 45, 2.0, True, True),
    ("exact_chebyshev_nojac_d6", "chebyshev", 1, 6, 24, 12, 6, 0, 46, 2.0, False, False),
    ("exact_fourier_d10", "fourier", 1, 8, 20, 9, 10, 0, 47, 1.5, True, True),
]


def make_kind_case(name, kind_s, exact, batch, d_in, d_out, degree, lut_size, seed, x_range, with_bias, jac):
    kind = BasisKind(kind_s)
    rng = np.random.default_rng(seed)
    k = feature_count(kind, degree)
    s = 1.0 / np.sqrt(d_in * k)
    x = rng.uniform(-x_range, x_range, size=(batch, d_in)).astype(np.float32)
    c_jod = rng.uniform(-s, s, size=(d_in, d_out, k)).astype(np.float32)
    dy = rng.standard_normal((batch, d_out)).astype(np.float32)
    bias = (0.01 * rng.standard_normal(d_out)).astype(np.float32) if with_bias else None
    coeff = CoeffTensor(d_in, d_out, k - 1, Layout.JOD, c_jod.astype(np.float64).reshape(-1))
    doj = reorder_to_doj(coeff)
    sched = TileSchedule.for_dims(d_in, d_out)
    path = BasisPath.EXACT_RECURRENCE if exact else BasisPath.LUT_INTERP
    mode = KernelMode(path, include_tanh_jacobian=bool(jac))
    lut = None if exact else lut_build(kind, degree, lut_size)
    b64 = None if bias is None else bias.astype(np.float64)
    y = fused_forward(x.astype(np.float64), doj, lut, sched, mode, b64, kind=kind)
    dc, dx = backward_fused(x.astype(np.float64), doj, dy.astype(np.float64), lut, sched, mode, kind=kind)
    out = dict(x=x, c_jod=c_jod, dy=dy, lut_size=np.int64(lut_size), degree=np.int64(degree),
               jacobian=np.int64(jac), kind=np.array(kind_s), exact=np.int64(exact),
               y=y, dc_doj=dc.as3d().copy(), dx=dx, db=dy.astype(np.float64).sum(axis=0))
    if bias is not None:
        out["bias"] = bias
    if exact and kind is CHEB:
        # the unfused reference kernels (kernels.py:450-510), trig and recurrence
        out["y_ref_trig"] = reference_forward(x.astype(np.float64), coeff, k - 1, trig=True)
        gt, xt = reference_backward(x.astype(np.float64), coeff, dy.astype(np.float64), trig=True,
                                    include_tanh_jacobian=bool(jac))
        out["dc_ref_trig_jod"] = gt.as3d().copy()
        out["dx_ref_trig"] = xt
    np.savez_compressed(HERE / f"kind_{name}.npz", **out)


def make_kind_luts():
    rng = np.random.default_rng(22)
    for kind_s, degree, n in (("legendre", 5, 1024), ("hermite", 6, 513), ("fourier", 3, 2048),
                              ("legendre", 12, 32768), ("fourier", 8, 4096)):
        kind = BasisKind(kind_s)
        tab = lut_build(kind, degree, n)
        grid = tab.grid()
        pts = np.concatenate([
            rng.uniform(-1.2, 1.2, 1000),
            grid[rng.integers(0, n, 100)],
            np.array([-1.0, 1.0, 0.0]),
        ]).astype(np.float32)
        vals, slopes = interp_rows_with_slope(tab, pts.astype(np.float64))
        cols = np.arange(0, n, 1 if n <= 4096 else 61)
        np.savez_compressed(
            HERE / f"lutk_{kind_s}_d{degree}_n{n}.npz",
            kind=np.array(kind_s), degree=np.int64(degree), lut_size=np.int64(n),
            cols=cols, values=tab.values[:, cols], slopes=tab.slopes[:, cols[cols < n - 1]],
            value_sums=tab.values.sum(axis=1), slope_sums=tab.slopes.astype(np.float64).sum(axis=1),
            step=np.float64(tab.step), points=pts, interp=vals, interp_slopes=slopes,
            bound=lut_max_error_bound(tab),
        )


def make_layer_case(name, batch, d_in, d_out, degree, lut_size, seed, x_range, with_bias, jac):
    rng = np.random.default_rng(seed)
    k = degree + 1
    s = 1.0 / np.sqrt(d_in * k)
    x = rng.uniform(-x_range, x_range, size=(batch, d_in)).astype(np.float32)
    c_jod = rng.uniform(-s, s, size=(d_in, d_out, k)).astype(np.float32)
    dy = rng.standard_normal((batch, d_out)).astype(np.float32)
    bias = (0.01 * rng.standard_normal(d_out)).astype(np.float32) if with_bias else None

    lut = lut_build(CHEB, degree, lut_size)
    coeff = CoeffTensor(d_in, d_out, degree, Layout.JOD, c_jod.astype(np.float64).reshape(-1))
    doj = reorder_to_doj(coeff)
    sched = TileSchedule.for_dims(d_in, d_out)
    mode = LUT_MODE if jac else KernelMode(BasisPath.LUT_INTERP, include_tanh_jacobian=False)
    y = fused_forward(x.astype(np.float64), doj, lut, sched, mode,
                      None if bias is None else bias.astype(np.float64))
    dc, dx = backward_fused(x.astype(np.float64), doj, dy.astype(np.float64), lut, sched, mode)
    db = dy.astype(np.float64).sum(axis=0)
    y_exact = reference_forward(x.astype(np.float64), coeff, degree, trig=True)
    if bias is not None:
        y_exact = y_exact + bias.astype(np.float64)
    out = dict(
        x=x, c_jod=c_jod, dy=dy, lut_size=np.int64(lut_size), degree=np.int64(degree),
        jacobian=np.int64(jac), y=y, dc_doj=dc.as3d().copy(), dx=dx, db=db, y_exact=y_exact,
    )
    if bias is not None:
        out["bias"] = bias
    np.savez_compressed(HERE / f"layer_{name}.npz", **out)


def make_lut_cases():
    # Known-answer tables (test_lut.py:29-33, 81-85, 96-99 pin these values).
    t = lut_build(CHEB, 2, 3)
    np.savez_compressed(HERE / "lut_kat_d2_n3.npz", values=t.values, slopes=t.slopes,
                        step=np.float64(t.step))
    # Interpolation of a float32 point cloud incl. clamps, nodes and cell edges.
    rng = np.random.default_rng(21)
    for degree, n in ((8, 1024), (8, 4096), (3, 512), (15, 16384), (5, 32768)):
        tab = lut_build(CHEB, degree, n)
        grid = tab.grid()
        pts = np.concatenate([
            rng.uniform(-1.2, 1.2, 1500),
            grid[rng.integers(0, n, 200)],              # node queries
            grid[rng.integers(0, n - 1, 200)] + tab.step * 0.5,  # cell midpoints
            np.array([-1.0, 1.0, -2.0, 3.0, 0.0]),
        ]).astype(np.float32)
        vals, slopes = interp_rows_with_slope(tab, pts.astype(np.float64))
        # Full tables only for small N; large ones keep every 61st column
        # plus exact per-feature sums (the oracle rebuilds and compares).
        cols = np.arange(0, n, 1 if n <= 4096 else 61)
        np.savez_compressed(
            HERE / f"lut_d{degree}_n{n}.npz",
            cols=cols, values=tab.values[:, cols], slopes=tab.slopes[:, cols[cols < n - 1]],
            value_sums=tab.values.sum(axis=1), slope_sums=tab.slopes.astype(np.float64).sum(axis=1),
            step=np.float64(tab.step),
            points=pts, interp=vals, interp_slopes=slopes,
            bound=lut_max_error_bound(tab),
        )


def main():
    HERE.mkdir(parents=True, exist_ok=True)
    make_lut_cases()
    for case in LAYER_CASES:
        make_layer_case(*case)
    make_kind_luts()
    for case in KIND_CASES:
        make_kind_case(*case)
    total = sum(p.stat().st_size for p in HERE.glob("*.npz"))
    print(f"wrote {len(list(HERE.glob('*.npz')))} fixtures, {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
