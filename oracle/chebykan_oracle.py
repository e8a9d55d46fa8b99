"""CPU oracle for the fused Chebyshev-KAN layer -- TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference's hot path
(arxiv 2511.14852 / PolyKAN, package ``polykan`` under
/root/reference/pkg/src/polykan): the LUT-interpolation and exact-recurrence
layer for all four basis families (Chebyshev, Legendre, Hermite, Fourier).  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product path
(``paper_2511_14852_b200``) never imports, links or calls anything here and
fails loudly when its CUDA library is missing.

Pinning: every function below is checked bit-for-bit (or to <=1e-13 where
BLAS summation order may differ) against golden vectors produced by running
the reference itself in the build container (``tests/golden/make_golden.py``
-> ``tests/golden/*.npz``; test ``tests/test_oracle_golden.py``).  The
trainer and file-format fixtures (``make_golden_train.py``,
``make_golden_formats.py``) pin the GPU model layer directly.

Citations are ``path:line`` relative to /root/reference/pkg/src/polykan/.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# lut.py:28 -- positions within this distance of a node snap onto it.
SNAP_EPS = 1e-9
# lut.py:32 -- the reference's default table size.
REFERENCE_DEFAULT_LUT_SIZE = 32768
# kernels.py:81-82 -- default CPU tile shape of TileSchedule.for_dims.
REF_TILE_IN = 64
REF_TILE_OUT = 32


# ---------------------------------------------------------------------------
# Basis and table construction


def chebyshev_rows(degree: int, t: np.ndarray) -> np.ndarray:
    """T_0..T_degree at every point by the three-term recurrence.

    basis.py:112-119 with the Chebyshev coefficients of basis.py:54-60
    (alpha=1, beta=2x, gamma=1); the division by alpha=1.0 is kept so the
    float64 rounding sequence is the reference's.
    """
    t = np.asarray(t, dtype=np.float64)
    rows = np.empty((degree + 1,) + t.shape, dtype=np.float64)
    rows[0] = np.ones_like(t)
    if degree >= 1:
        rows[1] = t.copy()
    for k in range(1, degree):
        rows[k + 1] = ((2.0 * t) * rows[k] - 1.0 * rows[k - 1]) / 1.0
    return rows


KINDS = ("chebyshev", "legendre", "hermite", "fourier")


def feature_count(kind: str, degree: int) -> int:
    """basis.py:24-34: Fourier has 2*degree+1 features, the others degree+1."""
    return 2 * degree + 1 if kind == "fourier" else degree + 1


def degree_for(kind: str, n_feat: int) -> int:
    """kernels.py:227-233."""
    return (n_feat - 1) // 2 if kind == "fourier" else n_feat - 1


def basis_rows(kind: str, degree: int, t: np.ndarray) -> np.ndarray:
    """All features at every point; basis.py:87-119 with the recurrence
    coefficients of basis.py:52-77 (alpha, beta(x), gamma), evaluated as
    (beta_k(x) * B_k - gamma_k * B_{k-1}) / alpha_k in numpy's order; Fourier
    by the angle-addition identities from cos/sin(pi x) (basis.py:100-110)."""
    if kind == "chebyshev":
        return chebyshev_rows(degree, t)
    t = np.asarray(t, dtype=np.float64)
    nf = feature_count(kind, degree)
    out = np.empty((nf,) + t.shape, dtype=np.float64)
    out[0] = 1.0
    if kind == "fourier":
        if degree >= 1:
            theta = np.pi * t
            c1, s1 = np.cos(theta), np.sin(theta)
            out[1], out[2] = c1, s1
            for k in range(1, degree):
                out[2 * k + 1] = c1 * out[2 * k - 1] - s1 * out[2 * k]
                out[2 * k + 2] = s1 * out[2 * k - 1] + c1 * out[2 * k]
        return out
    if degree >= 1:
        out[1] = 2.0 * t if kind == "hermite" else t.copy()
    for k in range(1, degree):
        if kind == "legendre":
            alpha, beta, gamma = float(k + 1), (2.0 * k + 1.0) * t, float(k)
        elif kind == "hermite":
            alpha, beta, gamma = 1.0, 2.0 * t, 2.0 * k
        else:
            raise ValueError(f"unsupported basis kind: {kind}")
        out[k + 1] = (beta * out[k] - gamma * out[k - 1]) / alpha
    return out


def derivative_rows(kind: str, degree: int, t: np.ndarray) -> np.ndarray:
    """Analytic dB_k/dx; basis.py:155-204 (T_n' = n U_{n-1}; P'_{k+1} =
    P'_{k-1} + (2k+1) P_k; H_n' = 2n H_{n-1}; d/dx of cos/sin(k pi x))."""
    t = np.asarray(t, dtype=np.float64)
    nf = feature_count(kind, degree)
    out = np.zeros((nf,) + t.shape, dtype=np.float64)
    if degree < 1:
        return out
    if kind == "chebyshev":
        u_prev = np.ones_like(t)
        out[1] = u_prev
        if degree >= 2:
            u_cur = 2.0 * t
            out[2] = 2.0 * u_cur
            for n in range(3, degree + 1):
                u_prev, u_cur = u_cur, 2.0 * t * u_cur - u_prev
                out[n] = n * u_cur
        return out
    b = basis_rows(kind, degree, t)
    if kind == "legendre":
        out[1] = 1.0
        for k in range(1, degree):
            out[k + 1] = out[k - 1] + (2.0 * k + 1.0) * b[k]
    elif kind == "hermite":
        for n in range(1, degree + 1):
            out[n] = 2.0 * n * b[n - 1]
    else:
        for k in range(1, degree + 1):
            kpi = k * np.pi
            out[2 * k - 1] = -kpi * b[2 * k]
            out[2 * k] = kpi * b[2 * k - 1]
    return out


def chebyshev_trig_rows(degree: int, t: np.ndarray) -> np.ndarray:
    """cos(k * arccos t), the exact path used for the interpolation report.

    basis.py:144-152.
    """
    t = np.asarray(t, dtype=np.float64)
    theta = np.arccos(t)
    k = np.arange(degree + 1, dtype=np.float64).reshape((degree + 1,) + (1,) * t.ndim)
    return np.cos(k * theta)


def build_table(degree: int, lut_size: int, kind: str = "chebyshev"):
    """Uniform-grid table of basis values (f64) and per-cell slopes (f32).

    lut.py:76-94: grid x_i = -1 + i*step with step = 2/(N-1) and the last
    node forced to exactly 1.0; slopes are float64 first differences over
    step, stored as float32.  Returns (values[K,N] f64, slopes[K,N-1] f32,
    step).
    """
    if lut_size < 2:
        raise ValueError("lut_size must be >= 2")
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    step = 2.0 / (lut_size - 1)
    nodes = -1.0 + step * np.arange(lut_size, dtype=np.float64)
    nodes[-1] = 1.0
    values = basis_rows(kind, degree, nodes)
    slopes = ((values[:, 1:] - values[:, :-1]) / step).astype(np.float32)
    return values, slopes, step


def interp_error_bound(degree: int, lut_size: int) -> np.ndarray:
    """Per-feature bound step^2/8 * max|T_k''| = step^2/8 * k^2 (k^2-1)/3.

    lut.py:143-153 (Chebyshev closed form, basis.py:215-217).
    """
    step = 2.0 / (lut_size - 1)
    k = np.arange(degree + 1, dtype=np.float64)
    return (step * step / 8.0) * np.maximum(k * k * (k * k - 1.0) / 3.0, 0.0)


def cell_positions(t: np.ndarray, lut_size: int):
    """Clamp to [-1,1], locate the cell, snap node echoes.  lut.py:97-106."""
    tc = np.clip(np.asarray(t, dtype=np.float64), -1.0, 1.0)
    pos = (tc + 1.0) * 0.5 * (lut_size - 1)
    idx = np.minimum(pos.astype(np.int64), lut_size - 2)
    frac = pos - idx
    frac = np.where(frac < SNAP_EPS, 0.0, frac)
    frac = np.where(frac > 1.0 - SNAP_EPS, 1.0, frac)
    return idx, frac


def lut_values(t: np.ndarray, values: np.ndarray) -> np.ndarray:
    """v[idx](1-f) + v[idx+1] f for every point; (...,) -> (..., K).

    lut.py:109-115 (the position-major copy of lut.py:64 is values.T).
    """
    idx, frac = cell_positions(t, values.shape[1])
    by_pos = np.ascontiguousarray(values.T)
    f = frac[..., None]
    return by_pos[idx] * (1.0 - f) + by_pos[idx + 1] * f


def lut_values_and_slopes(t: np.ndarray, values: np.ndarray, slopes: np.ndarray):
    """Interpolated values plus the active cell's float32 slope (as f64).

    lut.py:118-123 (slope copy lifted to f64 as in lut.py:66).
    """
    idx, frac = cell_positions(t, values.shape[1])
    by_pos = np.ascontiguousarray(values.T)
    s_by_pos = np.ascontiguousarray(slopes.T.astype(np.float64))
    f = frac[..., None]
    return by_pos[idx] * (1.0 - f) + by_pos[idx + 1] * f, s_by_pos[idx]


# ---------------------------------------------------------------------------
# Coefficient layouts (tensor.py:26-90)


def jod_to_doj(c_jod: np.ndarray) -> np.ndarray:
    """[I,O,K] -> contiguous [K,O,I]; tensor.py:77-82."""
    return np.ascontiguousarray(np.asarray(c_jod).transpose(2, 1, 0))


def doj_to_jod(c_doj: np.ndarray) -> np.ndarray:
    """[K,O,I] -> contiguous [I,O,K]; tensor.py:85-90."""
    return np.ascontiguousarray(np.asarray(c_doj).transpose(2, 1, 0))


# ---------------------------------------------------------------------------
# Fused LUT-mode layer


def _tiles(n: int, width: int):
    return [slice(s, min(s + width, n)) for s in range(0, n, width)]


def _run(fn, items, threads: int) -> None:
    # kernels.py:236-242: tasks own disjoint outputs, so order is irrelevant.
    if threads <= 1:
        for it in items:
            fn(it)
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(fn, items))


def _planes(t: np.ndarray, values: np.ndarray, slopes=None):
    """(K,B,I) contiguous basis planes (and slope planes); kernels.py:194-217."""
    if slopes is None:
        v = lut_values(t, values)
        return np.ascontiguousarray(v.transpose(2, 0, 1)), None
    v, s = lut_values_and_slopes(t, values, slopes)
    return (np.ascontiguousarray(v.transpose(2, 0, 1)),
            np.ascontiguousarray(s.transpose(2, 0, 1)))


def layer_forward(x, c_doj, values, bias=None, *, tile_in=REF_TILE_IN,
                  tile_out=REF_TILE_OUT, threads=1) -> np.ndarray:
    """y[b,o] = sum_i sum_k T_k(tanh x[b,i]) C[k,o,i] (+ bias[o]).

    Follows fused_forward (kernels.py:351-371): tanh (288), basis planes
    (289), per-(input tile, output tile) batched matmul summed over the
    order axis into a unique slot (293-318), then the combine stage folding
    input tiles in ascending order and adding the bias (321-348).
    """
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c_doj, dtype=np.float64)
    n_feat, d_out, d_in = c.shape
    if x.ndim != 2 or x.shape[1] != d_in:
        raise ValueError(f"input must be (batch, {d_in}), got {x.shape}")
    if values.shape[0] != n_feat:
        raise ValueError(f"LUT has {values.shape[0]} features, coefficients expect {n_feat}")
    batch = x.shape[0]
    planes, _ = _planes(np.tanh(x), values)
    return _tiled_forward(planes, c, bias, batch, tile_in, tile_out, threads)


def _tiled_forward(planes, c, bias, batch, tile_in, tile_out, threads):
    n_feat, d_out, d_in = c.shape
    ins, outs = _tiles(d_in, tile_in), _tiles(d_out, tile_out)
    partial = np.zeros((len(outs), len(ins), batch, tile_out))

    def task(pair):
        a, b = pair
        js, os_ = ins[a], outs[b]
        prod = np.matmul(planes[:, :, js], c[:, os_, js].swapaxes(1, 2))
        partial[b, a, :, : os_.stop - os_.start] = prod.sum(axis=0)

    _run(task, [(a, b) for a in range(len(ins)) for b in range(len(outs))], threads)
    y = np.zeros((batch, d_out))
    for b, os_ in enumerate(outs):
        acc = partial[b, 0, :, : os_.stop - os_.start].copy()
        for a in range(1, len(ins)):
            acc += partial[b, a, :, : os_.stop - os_.start]
        y[:, os_] = acc
    if bias is not None:
        y += np.asarray(bias, dtype=np.float64)
    return y


def layer_backward(x, c_doj, dy, values, slopes, *, include_tanh_jacobian=True,
                   tile_in=REF_TILE_IN, tile_out=REF_TILE_OUT, threads=1):
    """(dC in DOJ [K,O,I], dX [B,I], db [O]) for loss gradient dy.

    Follows backward_fused (kernels.py:374-447): per tile pair, dC tile =
    dy^T . planes (429); x-grad stage = sum_{k>=1} (dy . C_k) * slope_k
    (430-434); ordered merge over output tiles (439-442); tanh Jacobian
    (443-444).  db = dy.sum(0) is Layer.backward's bias gradient
    (model.py:147).
    """
    x = np.asarray(x, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    c = np.asarray(c_doj, dtype=np.float64)
    n_feat, d_out, d_in = c.shape
    batch = x.shape[0]
    if dy.shape != (batch, d_out):
        raise ValueError(f"dy must have shape ({batch}, {d_out}), got {dy.shape}")
    t = np.tanh(x)
    planes, slope_planes = _planes(t, values, slopes)
    return _tiled_backward(t, planes, slope_planes, c, dy, include_tanh_jacobian, tile_in, tile_out, threads)


def _tiled_backward(t, planes, slope_planes, c, dy, include_tanh_jacobian, tile_in, tile_out, threads):
    n_feat, d_out, d_in = c.shape
    batch = t.shape[0]
    ins, outs = _tiles(d_in, tile_in), _tiles(d_out, tile_out)
    dc = np.zeros_like(c)
    stage = np.zeros((len(outs), batch, d_in))

    def task(pair):
        a, b = pair
        js, os_ = ins[a], outs[b]
        dyt = dy[:, os_]
        dc[:, os_, js] = np.matmul(dyt.T[None, :, :], planes[:, :, js])
        if n_feat > 1:
            g = np.matmul(dyt[None, :, :], c[1:, os_, js])
            stage[b, :, js] = (g * slope_planes[1:, :, js]).sum(axis=0)

    _run(task, [(a, b) for a in range(len(ins)) for b in range(len(outs))], threads)
    dx = np.zeros((batch, d_in))
    for b in range(len(outs)):
        dx += stage[b]
    if include_tanh_jacobian:
        dx *= 1.0 - t * t
    return dc, dx, dy.sum(axis=0)


def exact_layer_forward(x, c_doj, kind: str = "chebyshev", bias=None, *, tile_in=REF_TILE_IN,
                        tile_out=REF_TILE_OUT, threads=1) -> np.ndarray:
    """fused_forward in EXACT_RECURRENCE mode (kernels.py:219-224): the same
    tiled contraction over basis_rows(kind, degree, tanh x)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c_doj, dtype=np.float64)
    planes = basis_rows(kind, degree_for(kind, c.shape[0]), np.tanh(x))
    return _tiled_forward(planes, c, bias, x.shape[0], tile_in, tile_out, threads)


def exact_layer_backward(x, c_doj, dy, kind: str = "chebyshev", *, include_tanh_jacobian=True,
                         tile_in=REF_TILE_IN, tile_out=REF_TILE_OUT, threads=1):
    """backward_fused in EXACT_RECURRENCE mode: planes = basis_rows, slope
    planes = derivative_rows at tanh x (kernels.py:222-224)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c_doj, dtype=np.float64)
    t = np.tanh(x)
    degree = degree_for(kind, c.shape[0])
    planes = basis_rows(kind, degree, t)
    deriv = derivative_rows(kind, degree, t)
    return _tiled_backward(t, planes, deriv, c, np.asarray(dy, dtype=np.float64), include_tanh_jacobian,
                           tile_in, tile_out, threads)


def exact_forward(x, c_doj, bias=None) -> np.ndarray:
    """Unfused exact cos(k acos tanh x) contraction; kernels.py:450-478 (trig=True)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c_doj, dtype=np.float64)
    planes = chebyshev_trig_rows(c.shape[0] - 1, np.tanh(x))
    y = np.einsum("kbi,koi->bo", planes, c)
    if bias is not None:
        y = y + bias
    return y


# ---------------------------------------------------------------------------
# Error measures


def max_rel_err(got, want, floor: float = 1e-9) -> float:
    """Elementwise relative error with a magnitude-aware floor; verify.py:45-57."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    big = float(np.abs(want).max(initial=0.0))
    scale = np.maximum(np.abs(want), max(floor, 1e-7 * big))
    return float(np.max(np.abs(got - want) / scale))


def normwise_err(got, want) -> float:
    """max|got-want| / max|want| -- the tolerance measure of SURVEY.md F1."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    big = float(np.abs(want).max(initial=0.0))
    return float(np.abs(got - want).max() / max(big, 1e-30))


# ---------------------------------------------------------------------------
# Seeded inputs (perf.py:157-169 distribution, generated in float32)


def bench_inputs(batch, d_in, d_out, degree, seed=0):
    """x ~ U(-1.5,1.5), C ~ U(-s,s) with s=1/sqrt(I*K) (JOD), dy ~ N(0,1).

    Mirrors perf.py:157-169 but draws in float32 so the GPU and the oracle
    see identical, exactly representable inputs.
    """
    rng = np.random.default_rng(seed)
    k = degree + 1
    s = 1.0 / math.sqrt(d_in * k)
    x = rng.uniform(-1.5, 1.5, size=(batch, d_in)).astype(np.float32)
    c_jod = rng.uniform(-s, s, size=(d_in, d_out, k)).astype(np.float32)
    dy = rng.standard_normal((batch, d_out)).astype(np.float32)
    return x, c_jod, dy


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)
