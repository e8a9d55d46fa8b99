"""Device-resident basis lookup tables (drop-in for polykan.lut).

Reference: /root/reference/pkg/src/polykan/lut.py.  ``lut_build(kind, degree,
lut_size)`` mirrors lut.py:76-94 (same grid, float64 recurrence, float32
slopes; bit-identical float64 values) and keeps float32 position-major
copies on the GPU for the kernels.  ``exact_basis`` is the table-free handle
of the exact evaluation path (BasisPath.EXACT_RECURRENCE, kernels.py:30-32).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .basis import BASIS_TAGS, CK_BASIS_CHEBYSHEV_TRIG, BasisKind, as_kind, feature_count

# lut.py:32 -- keep the reference default so an unmodified caller gets the
# same interpolation grid (and therefore identical results up to fp32/BF16x3
# round-off).
DEFAULT_LUT_SIZE = 32768


class _BasisHandle:
    """Owns a ``ck_lut`` handle of the C ABI (table or exact evaluation)."""

    exact = False

    def __init__(self, handle: int, kind: BasisKind, degree: int, device: int):
        self._handle = ctypes.c_void_p(handle)
        self.kind = kind
        self.degree = degree
        self.device = device
        nf = ctypes.c_int()
        _lib.check(_lib.lib().ck_lut_kind(self._handle, None, ctypes.byref(nf), None), "ck_lut_kind")
        self._n_feat = nf.value

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    @property
    def n_features(self) -> int:
        return self._n_feat

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                _lib.lib().ck_lut_destroy(h)
            except Exception:
                pass
            self._handle = None


class LutTable(_BasisHandle):
    """Sampled basis values plus per-cell slopes on one CUDA device (LutTable, lut.py:43-73).

    ``values`` / ``slopes`` read the table back as NumPy (float64 [K,N] /
    float32 [K,N-1]) for inspection and tests.
    """

    def __init__(self, handle: int, kind: BasisKind, degree: int, lut_size: int, device: int):
        super().__init__(handle, kind, degree, device)
        self.lut_size = lut_size
        step = ctypes.c_double()
        _lib.check(_lib.lib().ck_lut_info(self._handle, None, None, ctypes.byref(step)), "ck_lut_info")
        self.step = step.value

    def grid(self) -> np.ndarray:
        return -1.0 + self.step * np.arange(self.lut_size)

    def _read(self):
        v = np.empty((self.n_features, self.lut_size), dtype=np.float64)
        s = np.empty((self.n_features, self.lut_size - 1), dtype=np.float32)
        rc = _lib.lib().ck_lut_read(self._handle, v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    s.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        _lib.check(rc, "ck_lut_read")
        return v, s

    @property
    def values(self) -> np.ndarray:
        return self._read()[0]

    @property
    def slopes(self) -> np.ndarray:
        return self._read()[1]

    def __repr__(self) -> str:
        return (f"LutTable(kind={self.kind.value}, degree={self.degree}, lut_size={self.lut_size}, "
                f"device=cuda:{self.device})")


class ExactBasis(_BasisHandle):
    """Exact evaluation handle: the kernels evaluate basis_rows / derivative_rows at
    tanh(x) (basis.py:87-119, 155-204); ``trig`` selects cos(k acos t) for the
    Chebyshev values (trig_rows basis.py:144-152)."""

    exact = True

    def __init__(self, handle: int, kind: BasisKind, degree: int, device: int, trig: bool):
        super().__init__(handle, kind, degree, device)
        self.trig = trig

    def __repr__(self) -> str:
        return f"ExactBasis(kind={self.kind.value}, degree={self.degree}, trig={self.trig}, device=cuda:{self.device})"


def _device_index(device) -> int:
    import torch

    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"LutTable lives on a CUDA device, got {d}")
    return d.index if d.index is not None else torch.cuda.current_device()


def lut_build(kind: BasisKind, degree: int, lut_size: int = DEFAULT_LUT_SIZE, device=None) -> LutTable:
    """Sample every feature on the uniform grid and precompute cell slopes (lut.py:76-94)."""
    kind = as_kind(kind)
    if lut_size < 2:
        raise ValueError("lut_size must be >= 2")
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    dev = _device_index(device)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().ck_lut_build(BASIS_TAGS[kind], int(degree), int(lut_size), dev, ctypes.byref(h)),
               "ck_lut_build")
    return LutTable(h.value, kind, int(degree), int(lut_size), dev)


_EXACT_CACHE: dict = {}


def exact_basis(kind: BasisKind, degree: int, device=None, trig: bool = False) -> ExactBasis:
    """Table-free exact-evaluation handle (cached per kind/degree/device)."""
    kind = as_kind(kind)
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    if trig and kind is not BasisKind.CHEBYSHEV:
        raise ValueError("the trig path applies to the Chebyshev basis only")
    dev = _device_index(device)
    key = (kind, int(degree), dev, bool(trig))
    hit = _EXACT_CACHE.get(key)
    if hit is None:
        h = ctypes.c_void_p()
        code = CK_BASIS_CHEBYSHEV_TRIG if trig else BASIS_TAGS[kind]
        _lib.check(_lib.lib().ck_basis_exact(code, int(degree), dev, ctypes.byref(h)), "ck_basis_exact")
        hit = ExactBasis(h.value, kind, int(degree), dev, bool(trig))
        _EXACT_CACHE[key] = hit
    return hit


def lut_from_arrays(values: np.ndarray, slopes: np.ndarray, kind: BasisKind = BasisKind.CHEBYSHEV,
                    degree: int | None = None, device=None) -> LutTable:
    """Wrap caller-provided tables (e.g. a PKLT file read by load_lut, lut.py:180-206)."""
    kind = as_kind(kind)
    values = np.ascontiguousarray(values, dtype=np.float64)
    slopes = np.ascontiguousarray(slopes, dtype=np.float32)
    k, n = values.shape
    if slopes.shape != (k, n - 1):
        raise ValueError(f"slopes must have shape ({k}, {n - 1}), got {slopes.shape}")
    if degree is None:
        degree = (k - 1) // 2 if kind is BasisKind.FOURIER else k - 1
    if feature_count(kind, degree) != k:
        raise ValueError(f"{k} table rows do not match {kind.value} degree {degree}")
    dev = _device_index(device)
    h = ctypes.c_void_p()
    rc = _lib.lib().ck_lut_create(BASIS_TAGS[kind], int(degree), n,
                                  values.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  slopes.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), dev, ctypes.byref(h))
    _lib.check(rc, "ck_lut_create")
    return LutTable(h.value, kind, int(degree), n, dev)


def interp_error_bound(degree: int, lut_size: int) -> np.ndarray:
    """Chebyshev closed-form per-feature bound step^2/8 * k^2 (k^2-1)/3 (lut.py:143-153)."""
    step = 2.0 / (lut_size - 1)
    k = np.arange(degree + 1, dtype=np.float64)
    return (step * step / 8.0) * np.maximum(k * k * (k * k - 1.0) / 3.0, 0.0)


def _derivative_rows_host(kind: BasisKind, degree: int, x: np.ndarray) -> np.ndarray:
    """Analytic dB_k/dx on the host, only for the error-bound sampling below
    (derivative_rows semantics, basis.py:155-204)."""
    nf = feature_count(kind, degree)
    out = np.zeros((nf,) + x.shape)
    if kind is BasisKind.FOURIER:
        for k in range(1, degree + 1):
            out[2 * k - 1] = -k * np.pi * np.sin(k * np.pi * x)
            out[2 * k] = k * np.pi * np.cos(k * np.pi * x)
        return out
    v = np.empty((nf,) + x.shape)
    v[0] = 1.0
    if degree >= 1:
        v[1] = 2.0 * x if kind is BasisKind.HERMITE else x
    for k in range(1, degree):
        if kind is BasisKind.LEGENDRE:
            v[k + 1] = ((2 * k + 1) * x * v[k] - k * v[k - 1]) / (k + 1)
        elif kind is BasisKind.HERMITE:
            v[k + 1] = 2 * x * v[k] - 2 * k * v[k - 1]
        else:
            v[k + 1] = 2 * x * v[k] - v[k - 1]
    if kind is BasisKind.LEGENDRE:
        if degree >= 1:
            out[1] = 1.0
        for k in range(1, degree):
            out[k + 1] = out[k - 1] + (2 * k + 1) * v[k]
    elif kind is BasisKind.HERMITE:
        for n in range(1, degree + 1):
            out[n] = 2 * n * v[n - 1]
    else:
        u_prev, u_cur = np.ones_like(x), 2 * x
        if degree >= 1:
            out[1] = 1.0
        if degree >= 2:
            out[2] = 2 * u_cur
        for n in range(3, degree + 1):
            u_prev, u_cur = u_cur, 2 * x * u_cur - u_prev
            out[n] = n * u_cur
    return out


def lut_max_error_bound(table: LutTable) -> np.ndarray:
    """Per-feature interpolation-error bound step^2/8 * max|B_k''| (lut.py:143-162):
    Chebyshev closed form; other kinds by dense central differences of the
    analytic derivative with a 5 % margin, as the reference documents."""
    if table.kind is BasisKind.CHEBYSHEV:
        return interp_error_bound(table.degree, table.lut_size)
    lead = table.step * table.step / 8.0
    xs = np.linspace(-1.0, 1.0, 20001)
    h = 1e-5
    xs_in = np.clip(xs, -1.0 + h, 1.0 - h)
    d_plus = _derivative_rows_host(table.kind, table.degree, xs_in + h)
    d_minus = _derivative_rows_host(table.kind, table.degree, xs_in - h)
    curvature = np.abs((d_plus - d_minus) / (2.0 * h)).max(axis=1)
    return lead * curvature * 1.05


def lut_size_for_budget(degree: int, budget: float = 1e-4, cap: int = DEFAULT_LUT_SIZE) -> int:
    """Smallest power-of-two table whose closed-form bound is <= budget."""
    kmax = max(degree, 1)
    curv = kmax * kmax * (kmax * kmax - 1.0) / 3.0
    if curv <= 0:
        return 2
    need = 2.0 * math.sqrt(curv / (8.0 * budget)) + 1.0
    n = 2
    while n < need and n < cap:
        n *= 2
    return n


def expand(x, table, with_slopes: bool = False):
    """phi[..., k] = B_k(tanh x) by interpolation (+ cell slopes): interp_rows(_with_slope)
    (lut.py:109-123) applied to np.tanh(x) as in kernels.py:288/414.  With an
    ExactBasis: basis_rows / derivative_rows at tanh(x) (kernels.py:219-224)."""
    import torch

    if not x.is_cuda:
        raise ValueError("expand expects a CUDA tensor")
    xs = x.detach().to(torch.float32).contiguous()
    shape = xs.shape
    flat = xs.reshape(-1, shape[-1] if xs.dim() else 1)
    rows, cols = flat.shape
    phi = torch.empty(shape + (table.n_features,), device=x.device, dtype=torch.float32)
    slopes = torch.empty_like(phi) if with_slopes else None
    rc = _lib.lib().ck_expand(flat.data_ptr(), rows, cols, table.handle, phi.data_ptr(),
                              _lib.ptr(slopes), _lib.stream_handle(x.device))
    _lib.check(rc, "ck_expand")
    return (phi, slopes) if with_slopes else phi


# ---------------------------------------------------------------------------
# Interpolation at normalized points (no tanh), on the GPU (ck_basis_eval):
# interp_rows / interp_rows_with_slope / lut_interp / lut_interp_with_slope
# (lut.py:109-140) with the reference's float64 cell; float32 values.
# NumPy (or scalar) in -> NumPy out; torch CUDA tensors in -> torch out.


def _interp(table: LutTable, x, with_slope: bool):
    import torch

    is_torch = isinstance(x, torch.Tensor)
    xt = x.detach() if is_torch else torch.as_tensor(np.asarray(x, dtype=np.float64))
    dev = torch.device("cuda", table.device)
    flat = xt.to(device=dev, dtype=torch.float32).reshape(-1).contiguous()
    k = table.n_features
    vals = torch.empty((flat.numel(), k), dtype=torch.float32, device=dev)
    sl = torch.empty_like(vals) if with_slope else None
    _lib.check(_lib.lib().ck_basis_eval(flat.data_ptr(), flat.numel(), table.handle, vals.data_ptr(), _lib.ptr(sl),
                                        _lib.stream_handle(dev)), "ck_basis_eval")
    shape = tuple(xt.shape) + (k,)
    vals, sl = vals.reshape(shape), (None if sl is None else sl.reshape(shape))
    if not is_torch:
        vals = vals.cpu().numpy().astype(np.float64)
        sl = None if sl is None else sl.cpu().numpy().astype(np.float64)
    return (vals, sl) if with_slope else vals


def interp_rows(table: LutTable, x):
    """Interpolated feature values; (...,) -> (..., n_features) (lut.py:109-115)."""
    return _interp(table, x, False)


def interp_rows_with_slope(table: LutTable, x):
    """Values plus the active cell's slope per feature (lut.py:118-123)."""
    return _interp(table, x, True)


def lut_interp(table: LutTable, x: float):
    """Approximate feature vector at one point (lut.py:126-131)."""
    if not np.all(np.isfinite(np.asarray(x, dtype=np.float64))):
        raise ValueError("lut_interp requires finite input")
    return _interp(table, np.asarray(x, dtype=np.float64).reshape(1), False)[0]


def lut_interp_with_slope(table: LutTable, x: float):
    """Values and the piecewise-constant surrogate derivative at one point (lut.py:134-140)."""
    if not np.all(np.isfinite(np.asarray(x, dtype=np.float64))):
        raise ValueError("lut_interp_with_slope requires finite input")
    v, s = _interp(table, np.asarray(x, dtype=np.float64).reshape(1), True)
    return v[0], s[0]
