"""Basis families of the KAN layer (drop-in for polykan.basis's public enum).

Reference: /root/reference/pkg/src/polykan/basis.py.  ``BasisKind`` keeps the
reference's member names and values (basis.py:17-21) and ``feature_count``
its rule (basis.py:24-34).  The evaluation itself (recurrences, derivatives,
cos(k acos t)) runs on the device: the table build in the library's float64
builder, the expansion and the input-gradient epilogue in the sm_100a
kernels (csrc/ck_basis.cuh).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Callable


class BasisKind(Enum):
    CHEBYSHEV = "chebyshev"
    LEGENDRE = "legendre"
    HERMITE = "hermite"
    FOURIER = "fourier"


@dataclass(frozen=True)
class RecurrenceCoeffs:
    """alpha_k B_{k+1} = beta_k(x) B_k - gamma_k B_{k-1} with seeds (basis.py:37-49).
    The data the table builder and the kernels' recurrences implement."""

    alpha_k: Callable[[int], float]
    beta_k: Callable
    gamma_k: Callable[[int], float]
    seed0: Callable
    seed1: Callable


RECURRENCES = {  # basis.py:52-77
    BasisKind.CHEBYSHEV: RecurrenceCoeffs(lambda k: 1.0, lambda k, x: 2.0 * x, lambda k: 1.0,
                                          lambda x: x * 0 + 1.0, lambda x: x * 1.0),
    BasisKind.LEGENDRE: RecurrenceCoeffs(lambda k: float(k + 1), lambda k, x: (2.0 * k + 1.0) * x,
                                         lambda k: float(k), lambda x: x * 0 + 1.0, lambda x: x * 1.0),
    BasisKind.HERMITE: RecurrenceCoeffs(lambda k: 1.0, lambda k, x: 2.0 * x, lambda k: 2.0 * k,
                                        lambda x: x * 0 + 1.0, lambda x: 2.0 * x),
}

# ck_basis_kind codes (include/chebykan.h) == the PKLT basis tags (lut.py:35-40)
BASIS_TAGS = {
    BasisKind.CHEBYSHEV: 0,
    BasisKind.LEGENDRE: 1,
    BasisKind.HERMITE: 2,
    BasisKind.FOURIER: 3,
}
TAG_TO_BASIS = {v: k for k, v in BASIS_TAGS.items()}
# exact-only cos(k acos t) evaluation (trig_rows basis.py:144-152)
CK_BASIS_CHEBYSHEV_TRIG = 4


def as_kind(kind) -> BasisKind:
    """BasisKind from a BasisKind, its value string or its tag."""
    if isinstance(kind, BasisKind):
        return kind
    if isinstance(kind, str):
        return BasisKind(kind)
    if isinstance(kind, int) and kind in TAG_TO_BASIS:
        return TAG_TO_BASIS[kind]
    raise ValueError(f"unsupported basis kind: {kind!r}")


def feature_count(kind: BasisKind, degree: int) -> int:
    """degree + 1 features, or 2*degree + 1 for Fourier (basis.py:24-34)."""
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    if as_kind(kind) is BasisKind.FOURIER:
        return 2 * degree + 1
    return degree + 1


def degree_for(kind: BasisKind, n_feat: int) -> int:
    """Inverse of feature_count (kernels.py:227-233)."""
    if as_kind(kind) is BasisKind.FOURIER:
        if n_feat % 2 == 0:
            raise ValueError("Fourier feature count must be odd (2 * degree + 1)")
        return (n_feat - 1) // 2
    return n_feat - 1


def parse_kind(name: str) -> BasisKind:
    """basis.py:220-225."""
    try:
        return BasisKind(name.lower())
    except ValueError:
        valid = ", ".join(k.value for k in BasisKind)
        raise ValueError(f"unknown basis {name!r}; expected one of: {valid}") from None


def chebyshev_second_derivative_max(k: int) -> float:
    """max over [-1,1] of |T_k''| = k^2 (k^2 - 1) / 3 (basis.py:215-217)."""
    return k * k * (k * k - 1) / 3.0


# ---------------------------------------------------------------------------
# Point evaluation on the GPU (ck_basis_eval on an exact-evaluation handle):
# the reference's basis_rows / derivative_rows / trig_rows / eval_basis*
# (basis.py:87-212) in float32.  NumPy in -> NumPy out (float64 dtype holding
# float32 values); torch CUDA tensors in -> torch out.


def _eval(kind, degree: int, x, trig: bool, want_deriv: bool):
    import numpy as np
    import torch

    from . import _lib
    from .lut import exact_basis

    kind = as_kind(kind)
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    is_torch = isinstance(x, torch.Tensor)
    xt = x.detach() if is_torch else torch.as_tensor(np.asarray(x, dtype=np.float64))
    if not bool(torch.isfinite(xt).all()):
        raise ValueError("basis evaluation requires finite inputs")
    if trig and bool((xt.abs() > 1.0).any()):
        raise ValueError("trig evaluation requires |x| <= 1")
    dev = xt.device if (is_torch and xt.is_cuda) else torch.device("cuda", torch.cuda.current_device())
    flat = xt.to(device=dev, dtype=torch.float32).reshape(-1).contiguous()
    h = exact_basis(kind, degree, device=dev, trig=trig)
    k = h.n_features
    vals = torch.empty((flat.numel(), k), dtype=torch.float32, device=dev)
    der = torch.empty_like(vals) if want_deriv else None
    rc = _lib.lib().ck_basis_eval(flat.data_ptr(), flat.numel(), h.handle, vals.data_ptr(), _lib.ptr(der),
                                  _lib.stream_handle(dev))
    _lib.check(rc, "ck_basis_eval")
    out = (der if want_deriv else vals).t().reshape((k,) + tuple(xt.shape))
    if is_torch:
        return out
    return out.cpu().numpy().astype(np.float64)


def basis_rows(kind: BasisKind, degree: int, x):
    """All features at each point; shape (n_features,) + x.shape (basis.py:87-119)."""
    return _eval(kind, degree, x, False, False)


def derivative_rows(kind: BasisKind, degree: int, x):
    """Analytic derivatives dB_k/dx; shape (n_features,) + x.shape (basis.py:155-204)."""
    return _eval(kind, degree, x, False, True)


def trig_rows(degree: int, x):
    """cos(n arccos x), shape (degree+1,) + x.shape (basis.py:144-152)."""
    return _eval(BasisKind.CHEBYSHEV, degree, x, True, False)


def _scalar(x, what: str):
    import numpy as np

    xv = np.asarray(x, dtype=np.float64)
    if xv.ndim != 0:
        raise ValueError(what)
    return xv.reshape(1)


def eval_basis(kind: BasisKind, degree: int, x: float):
    """Feature vector [B_0(x), ..., B_d(x)] at one normalized point (basis.py:122-128)."""
    return basis_rows(kind, degree, _scalar(x, "eval_basis takes a scalar; use basis_rows for arrays"))[:, 0]


def eval_basis_trig(degree: int, x: float):
    """Chebyshev values via cos(n arccos x) at one point (basis.py:131-141)."""
    return trig_rows(degree, _scalar(x, "eval_basis_trig takes a scalar"))[:, 0]


def eval_basis_derivative(kind: BasisKind, degree: int, x: float):
    """Analytic derivative vector at one point (basis.py:205-210)."""
    return derivative_rows(kind, degree, _scalar(x, "eval_basis_derivative takes a scalar"))[:, 0]
