"""Device-resident Chebyshev lookup tables (drop-in for polykan.lut).

Reference: /root/reference/pkg/src/polykan/lut.py.  ``lut_build`` mirrors
lut.py:76-94 (same grid, float64 recurrence, float32 slopes) but builds the
table on the GPU (bit-identical float64 values) and keeps float32
position-major copies there for the kernels.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

# lut.py:32 -- keep the reference default so an unmodified caller gets the
# same interpolation grid (and therefore identical results up to fp32/BF16x3
# round-off).  Smaller tables trade interpolation error for shared-memory
# residency; see interp_error_bound.
DEFAULT_LUT_SIZE = 32768


class LutTable:
    """Chebyshev LUT on one CUDA device (LutTable, lut.py:43-73).

    Owns a ``ck_lut`` handle.  ``values`` / ``slopes`` read the table back as
    NumPy (float64 [K,N] / float32 [K,N-1]) for inspection and tests.
    """

    kind = "chebyshev"

    def __init__(self, handle: int, degree: int, lut_size: int, device: int):
        self._handle = ctypes.c_void_p(handle)
        self.degree = degree
        self.lut_size = lut_size
        self.device = device
        step = ctypes.c_double()
        _lib.check(_lib.lib().ck_lut_info(self._handle, None, None, ctypes.byref(step)), "ck_lut_info")
        self.step = step.value

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    @property
    def n_features(self) -> int:
        return self.degree + 1

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

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                _lib.lib().ck_lut_destroy(h)
            except Exception:
                pass
            self._handle = None

    def __repr__(self) -> str:
        return f"LutTable(degree={self.degree}, lut_size={self.lut_size}, device=cuda:{self.device})"


def _device_index(device) -> int:
    import torch

    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"LutTable lives on a CUDA device, got {d}")
    return d.index if d.index is not None else torch.cuda.current_device()


def lut_build(degree: int, lut_size: int = DEFAULT_LUT_SIZE, device=None) -> LutTable:
    """Build the Chebyshev table on the GPU (lut_build, lut.py:76-94).

    The reference's ``kind`` argument is fixed to Chebyshev here (the only
    basis on this hot path).
    """
    if lut_size < 2:
        raise ValueError("lut_size must be >= 2")
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    dev = _device_index(device)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().ck_lut_build(int(degree), int(lut_size), dev, ctypes.byref(h)), "ck_lut_build")
    return LutTable(h.value, int(degree), int(lut_size), dev)


def lut_from_arrays(values: np.ndarray, slopes: np.ndarray, device=None) -> LutTable:
    """Wrap caller-provided tables (e.g. a PKLT file read by load_lut, lut.py:180-206)."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    slopes = np.ascontiguousarray(slopes, dtype=np.float32)
    k, n = values.shape
    if slopes.shape != (k, n - 1):
        raise ValueError(f"slopes must have shape ({k}, {n - 1}), got {slopes.shape}")
    dev = _device_index(device)
    h = ctypes.c_void_p()
    rc = _lib.lib().ck_lut_create(k - 1, n, values.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  slopes.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), dev, ctypes.byref(h))
    _lib.check(rc, "ck_lut_create")
    return LutTable(h.value, k - 1, n, dev)


def interp_error_bound(degree: int, lut_size: int) -> np.ndarray:
    """Closed-form per-feature bound step^2/8 * k^2 (k^2-1)/3 (lut.py:143-153)."""
    step = 2.0 / (lut_size - 1)
    k = np.arange(degree + 1, dtype=np.float64)
    return (step * step / 8.0) * np.maximum(k * k * (k * k - 1.0) / 3.0, 0.0)


def lut_max_error_bound(table: LutTable) -> np.ndarray:
    return interp_error_bound(table.degree, table.lut_size)


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


def expand(x, table: LutTable, with_slopes: bool = False):
    """phi[..., k] = T_k(tanh x) by interpolation (+ cell slopes): interp_rows(_with_slope)
    (lut.py:109-123) applied to np.tanh(x) as in kernels.py:288/414."""
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
