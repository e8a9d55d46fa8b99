"""Basis families of the KAN layer (drop-in for polykan.basis's public enum).

Reference: /root/reference/pkg/src/polykan/basis.py.  ``BasisKind`` keeps the
reference's member names and values (basis.py:17-21) and ``feature_count``
its rule (basis.py:24-34).  The evaluation itself (recurrences, derivatives,
cos(k acos t)) runs on the device: the table build in the library's float64
builder, the expansion and the input-gradient epilogue in the sm_100a
kernels (csrc/ck_basis.cuh).
"""
from __future__ import annotations

from enum import Enum


class BasisKind(Enum):
    CHEBYSHEV = "chebyshev"
    LEGENDRE = "legendre"
    HERMITE = "hermite"
    FOURIER = "fourier"


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
