"""On-disk interchange formats of the reference, byte-compatible.

* PKLT lookup tables (lut.py:165-206): magic, version u32, basis tag u8,
  degree u32, lut_size u32, then float32 values [K][N] and slopes [K][N-1].
* PKCK coefficient tensors (tensor.py:93-126): magic, version, layout tag,
  d_in, d_out, degree as u32, then the float32 payload in the tagged layout.
* PKMX matrices (cli.py:59-82): magic, version, rows, cols as u32, float32
  row-major -- the file boundary of ``polykan apply`` that the reference's
  TypeScript binding drives (pkg/frontend/src/layer.ts:173-261).

All fields little-endian.  Readers raise ValueError with the reference's
messages.  Tables load straight onto the GPU (``load_lut``); coefficient
and matrix payloads load as float64 CPU tensors like the reference's
float64 lift, and the layer entry points move them to the device.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .basis import BASIS_TAGS, TAG_TO_BASIS, feature_count
from .lut import LutTable, lut_from_arrays
from .tensor import CoeffTensor, Layout

LUT_MAGIC = b"PKLT"
LUT_VERSION = 1
COEFF_MAGIC = b"PKCK"
COEFF_VERSION = 1
MATRIX_MAGIC = b"PKMX"
MATRIX_VERSION = 1

_LAYOUT_TAGS = {Layout.JOD: 0, Layout.DOJ: 1}
_TAG_TO_LAYOUT = {v: k for k, v in _LAYOUT_TAGS.items()}


def _np(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


# --- PKLT (lut.py:165-206) ----------------------------------------------------

def save_lut(table: LutTable, path: str | Path) -> None:
    """Write the PKLT binary; float32 payload (lut.py:165-177)."""
    header = LUT_MAGIC + struct.pack("<IBII", LUT_VERSION, BASIS_TAGS[table.kind], table.degree, table.lut_size)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(table.values, dtype="<f4").tobytes())
        fh.write(np.ascontiguousarray(table.slopes, dtype="<f4").tobytes())


def read_lut_arrays(path: str | Path):
    """(kind, degree, lut_size, values f64 [K,N], slopes f32 [K,N-1]) of a PKLT file (lut.py:180-206)."""
    raw = Path(path).read_bytes()
    if raw[:4] != LUT_MAGIC:
        raise ValueError(f"{path}: not a PKLT file")
    version, tag, degree, lut_size = struct.unpack("<IBII", raw[4:17])
    if version != LUT_VERSION:
        raise ValueError(f"{path}: unsupported PKLT version {version}")
    if tag not in TAG_TO_BASIS:
        raise ValueError(f"{path}: unknown basis tag {tag}")
    kind = TAG_TO_BASIS[tag]
    nfeat = feature_count(kind, degree)
    n_values = nfeat * lut_size
    n_slopes = nfeat * (lut_size - 1)
    expected = 17 + 4 * (n_values + n_slopes)
    if len(raw) != expected:
        raise ValueError(f"{path}: expected {expected} bytes, found {len(raw)}")
    values = np.frombuffer(raw, dtype="<f4", count=n_values, offset=17)
    slopes = np.frombuffer(raw, dtype="<f4", count=n_slopes, offset=17 + 4 * n_values)
    return (kind, degree, lut_size, values.reshape(nfeat, lut_size).astype(np.float64),
            slopes.reshape(nfeat, lut_size - 1).copy())


def load_lut(path: str | Path, device=None) -> LutTable:
    """Read a PKLT file onto the GPU; values lifted to float64 (lut.py:180-206)."""
    kind, degree, _, values, slopes = read_lut_arrays(path)
    return lut_from_arrays(values, slopes, kind=kind, degree=degree, device=device)


# --- PKCK (tensor.py:93-126) --------------------------------------------------

def save_coeff(c: CoeffTensor, path: str | Path) -> None:
    """Write the PKCK binary with a float32 payload in the tagged layout."""
    header = COEFF_MAGIC + struct.pack("<IIIII", COEFF_VERSION, _LAYOUT_TAGS[c.layout], c.d_in, c.d_out, c.degree)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(_np(c.data), dtype="<f4").tobytes())


def load_coeff(path: str | Path) -> CoeffTensor:
    """Read a PKCK file; payload lifted to float64 (CPU tensor)."""
    raw = Path(path).read_bytes()
    if raw[:4] != COEFF_MAGIC:
        raise ValueError(f"{path}: not a PKCK file")
    version, tag, d_in, d_out, degree = struct.unpack("<IIIII", raw[4:24])
    if version != COEFF_VERSION:
        raise ValueError(f"{path}: unsupported PKCK version {version}")
    if tag not in _TAG_TO_LAYOUT:
        raise ValueError(f"{path}: unknown layout tag {tag}")
    count = d_in * d_out * (degree + 1)
    if len(raw) != 24 + 4 * count:
        raise ValueError(f"{path}: expected {24 + 4 * count} bytes, found {len(raw)}")
    data = np.frombuffer(raw, dtype="<f4", count=count, offset=24).astype(np.float64)
    return CoeffTensor(d_in, d_out, degree, _TAG_TO_LAYOUT[tag], torch.from_numpy(data))


# --- PKMX (cli.py:59-82) ------------------------------------------------------

def save_matrix(arr, path: str | Path) -> None:
    """Little-endian float32 matrix interchange file."""
    a = _np(arr)
    if a.ndim != 2:
        raise ValueError(f"matrix files hold 2-D data, got shape {a.shape}")
    with open(path, "wb") as fh:
        fh.write(MATRIX_MAGIC)
        fh.write(struct.pack("<III", MATRIX_VERSION, a.shape[0], a.shape[1]))
        fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_matrix(path: str | Path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if raw[:4] != MATRIX_MAGIC:
        raise ValueError(f"{path}: not a PKMX matrix file")
    version, rows, cols = struct.unpack("<III", raw[4:16])
    if version != MATRIX_VERSION:
        raise ValueError(f"{path}: unsupported PKMX version {version}")
    if len(raw) != 16 + 4 * rows * cols:
        raise ValueError(f"{path}: expected {16 + 4 * rows * cols} bytes, found {len(raw)}")
    return np.frombuffer(raw, dtype="<f4", count=rows * cols, offset=16).reshape(rows, cols).astype(np.float64)
