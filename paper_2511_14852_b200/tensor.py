"""Coefficient tensors with explicit layout tags (drop-in for polykan.tensor).

Reference: /root/reference/pkg/src/polykan/tensor.py.  JOD = [input, output,
order] (tensor.py:26-28, the original ChebyKAN ``cheby_coeffs`` shape); DOJ =
[order, output, input], unit stride in the input index -- the layout the
forward kernel streams with TMA.  Data are torch tensors (any device).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch


class Layout(Enum):
    JOD = "jod"
    DOJ = "doj"


@dataclass
class CoeffTensor:
    """Dense coefficients; ``data`` is contiguous in the tagged layout (tensor.py:31-64)."""

    d_in: int
    d_out: int
    degree: int
    layout: Layout
    data: torch.Tensor

    def __post_init__(self) -> None:
        if self.d_in < 1 or self.d_out < 1:
            raise ValueError("d_in and d_out must be >= 1")
        if self.degree < 0:
            raise ValueError("degree must be >= 0")
        expected = self.d_in * self.d_out * (self.degree + 1)
        if self.data.numel() != expected:
            raise ValueError(f"data has {self.data.numel()} entries, expected {expected}")
        self.data = self.data.reshape(self.shape3d()).contiguous()

    @property
    def n_feat(self) -> int:
        return self.degree + 1

    def shape3d(self):
        if self.layout is Layout.JOD:
            return (self.d_in, self.d_out, self.n_feat)
        return (self.n_feat, self.d_out, self.d_in)

    def as3d(self) -> torch.Tensor:
        return self.data.reshape(self.shape3d())


def jod_index(d_out: int, degree: int, j: int, o: int, k: int) -> int:
    """Flat offset of (j, o, k) in JOD (tensor.py:67-69)."""
    return (j * d_out + o) * (degree + 1) + k


def doj_index(d_in: int, d_out: int, k: int, o: int, j: int) -> int:
    """Flat offset of (k, o, j) in DOJ, unit stride along j (tensor.py:72-74)."""
    return (k * d_out + o) * d_in + j


def reorder_to_doj(c: CoeffTensor) -> CoeffTensor:
    """Physical copy JOD -> DOJ (tensor.py:77-82)."""
    if c.layout is not Layout.JOD:
        raise ValueError(f"reorder_to_doj expects JOD input, got {c.layout.value}")
    return CoeffTensor(c.d_in, c.d_out, c.degree, Layout.DOJ, c.as3d().permute(2, 1, 0).contiguous())


def reorder_to_jod(c: CoeffTensor) -> CoeffTensor:
    """Physical copy DOJ -> JOD (tensor.py:85-90)."""
    if c.layout is not Layout.DOJ:
        raise ValueError(f"reorder_to_jod expects DOJ input, got {c.layout.value}")
    return CoeffTensor(c.d_in, c.d_out, c.degree, Layout.JOD, c.as3d().permute(2, 1, 0).contiguous())
