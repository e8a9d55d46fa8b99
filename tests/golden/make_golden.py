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

from polykan.basis import BasisKind
from polykan.kernels import (
    BasisPath,
    KernelMode,
    LUT_MODE,
    TileSchedule,
    backward_fused,
    fused_forward,
    reference_forward,
)
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
    total = sum(p.stat().st_size for p in HERE.glob("*.npz"))
    print(f"wrote {len(list(HERE.glob('*.npz')))} fixtures, {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
