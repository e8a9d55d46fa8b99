"""ChebyKAN layer as a torch module with an autograd Function over the C ABI.

Drop-in for the reference's ``Layer`` (model.py:86-148): constructor
(input_dim, output_dim, degree), coefficients held in DOJ for the model's
lifetime (model.py:97-101), seeded U(-s, s) init with s = 1/sqrt(I*K)
(model.py:72-83), zero bias, forward caching x, backward returning dC, db,
dX.  Leading dimensions are flattened like nn.Linear (the speech model feeds
[batch, frames, bins]).
"""
from __future__ import annotations

import math

import numpy as np
import torch
from torch import nn

from .basis import BasisKind, as_kind, feature_count
from .kernels import BasisPath, PreparedCoeff, backward_raw, basis_cache_bytes, forward_raw
from .lut import DEFAULT_LUT_SIZE, exact_basis, lut_build


class _LayerState:
    """Per-module basis handle (LUT or exact) and coefficient-prep cache (not a parameter)."""

    def __init__(self, kind: BasisKind, degree: int, lut_size: int, jacobian: bool, exact: bool,
                 cache_basis="auto"):
        self.kind = kind
        self.degree = degree
        self.lut_size = lut_size
        self.jacobian = jacobian
        self.exact = exact
        self.cache_basis = cache_basis
        self._luts: dict = {}
        self._prep: PreparedCoeff | None = None
        self.grad_sink = None  # set by a data-parallel reducer's bind() (parallel.py)

    def lut(self, device: torch.device):
        idx = device.index if device.index is not None else torch.cuda.current_device()
        t = self._luts.get(idx)
        if t is None:
            dev = torch.device("cuda", idx)
            if self.exact:
                t = exact_basis(self.kind, self.degree, device=dev)
            else:
                t = lut_build(self.kind, self.degree, self.lut_size, device=dev)
            self._luts[idx] = t
        return t

    def prepared(self, coeff_doj: torch.Tensor) -> PreparedCoeff:
        """The bf16 operands of the current coefficients, re-split when the
        parameter changed.  Change detection is the tensor's storage, address
        and autograd version counter; writes that bypass the counter
        (``param.data.copy_()``, raw-pointer kernels) need invalidate()."""
        p = self._prep
        if p is None or p.device != coeff_doj.device or tuple(coeff_doj.shape) != (p.n_feat, p.d_out, p.d_in):
            p = PreparedCoeff(coeff_doj)
            self._prep = p
        elif p.key != PreparedCoeff.key_of(coeff_doj):
            p.update(coeff_doj)
        return p

    def invalidate(self) -> None:
        if self._prep is not None:
            self._prep.key = None


_TOTAL_MEM: dict = {}


def _free_bytes_estimate(device: torch.device) -> int:
    """Device memory not held by this process's tensors -- host-side counters
    only (cudaMemGetInfo synchronises and stalls behind other GPU clients)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    total = _TOTAL_MEM.get(idx)
    if total is None:
        total = _TOTAL_MEM[idx] = torch.cuda.get_device_properties(idx).total_memory
    return total - torch.cuda.memory_allocated(idx)


class ChebyKANFunction(torch.autograd.Function):
    """y = ChebyKAN(x; C, b).  Forward: ck_forward.  Backward: ck_backward."""

    @staticmethod
    def forward(ctx, x, coeff_doj, bias, state: _LayerState, want_cache: bool = False):
        if not x.is_cuda:
            raise ValueError("ChebyKAN kernels run on CUDA tensors only (no CPU fallback)")
        x = x.to(torch.float32).contiguous()
        lut = state.lut(x.device)
        prep = state.prepared(coeff_doj)
        cache = None
        # (ctx.needs_input_grad says True for a Parameter even under no_grad:
        # the caller decides, so inference never fills a basis cache and
        # narrow layers keep the shared-memory generated forward)
        if want_cache and state.cache_basis:
            # keep the expanded basis for dC (saves the backward's re-expansion)
            nbytes = basis_cache_bytes(x.shape[0], prep.d_in, prep.d_out, prep.n_feat)
            if nbytes > 0 and (state.cache_basis is True or nbytes <= 0.35 * _free_bytes_estimate(x.device)):
                cache = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        y = forward_raw(x, prep, lut, None if bias is None else bias.detach(), cache)
        ctx.save_for_backward(x, coeff_doj)
        ctx.state = state
        ctx.cache = cache
        ctx.has_bias = bias is not None
        return y

    @staticmethod
    def backward(ctx, dy):
        x, coeff_doj = ctx.saved_tensors
        state: _LayerState = ctx.state
        dy = dy.to(torch.float32).contiguous()
        need_x, need_c, need_b = ctx.needs_input_grad[0], ctx.needs_input_grad[1], ctx.needs_input_grad[2]
        prep = state.prepared(coeff_doj)
        # data-parallel binding (parallel.py): dC / db straight into the
        # exchange buffer, and the exchange started on its grads-ready event
        sink = state.grad_sink if need_c else None
        outs = sink.try_begin() if sink is not None else None
        dc_out, db_out, ev = outs if outs is not None else (None, None, None)
        dc, dx, db = backward_raw(x, dy, prep, state.lut(x.device), state.jacobian, want_dx=need_x,
                                  want_dc=need_c, want_db=need_b and ctx.has_bias, cache=ctx.cache,
                                  dc_out=dc_out, db_out=db_out if need_b and ctx.has_bias else None, grads_ready=ev)
        if outs is not None:
            sink.done()
        ctx.cache = None
        return dx, dc, db, None, None


class ChebyKANLayer(nn.Module):
    """Chebyshev-KAN layer y = sum_i sum_k C[k,o,i] T_k(tanh x_i) + b_o (or any
    basis family of the reference: ``kind``).

    Parameters
    ----------
    input_dim, output_dim, degree : layer shape (LayerSpec, model.py:37-54)
    kind : basis family (BasisKind, basis.py:17-21; default Chebyshev); the
        layer has feature_count(kind, degree) coefficient planes
    basis_path : BasisPath.LUT_INTERP (table, default) or EXACT_RECURRENCE
    bias : learnable bias, zero-initialised (model.py:82)
    lut_size : interpolation table size (reference default 32768, lut.py:32)
    include_tanh_jacobian : KernelMode flag (kernels.py:35-44)
    seed : when given, coefficients are drawn exactly as init_params
        (numpy default_rng(seed).uniform(-s, s) in JOD order, model.py:72-83)
    cache_basis : keep the forward's expanded basis (bf16 hi/lo planes,
        4*B*I*degree bytes) for the coefficient-gradient GEMM: "auto" when it
        fits in 35 % of free device memory, True, or False (re-expand)
    """

    def __init__(self, input_dim: int, output_dim: int, degree: int, bias: bool = True,
                 lut_size: int = DEFAULT_LUT_SIZE, include_tanh_jacobian: bool = True, seed: int | None = None,
                 device=None, cache_basis="auto", kind: BasisKind = BasisKind.CHEBYSHEV,
                 basis_path: BasisPath = BasisPath.LUT_INTERP):
        super().__init__()
        if input_dim < 1 or output_dim < 1:
            raise ValueError("layer dimensions must be >= 1")
        if degree < 0:
            raise ValueError("degree must be >= 0")
        self.input_dim, self.output_dim, self.degree = int(input_dim), int(output_dim), int(degree)
        self.lut_size = int(lut_size)
        self.kind = as_kind(kind)
        self.basis_path = BasisPath(basis_path)
        self.include_tanh_jacobian = bool(include_tanh_jacobian)
        k = feature_count(self.kind, self.degree)
        self.coeff_doj = nn.Parameter(torch.empty((k, self.output_dim, self.input_dim), device=device))
        self.bias = nn.Parameter(torch.zeros(self.output_dim, device=device)) if bias else None
        self._state = _LayerState(self.kind, self.degree, self.lut_size, self.include_tanh_jacobian,
                                  self.basis_path is BasisPath.EXACT_RECURRENCE, cache_basis)
        self.reset_parameters(seed)

    @property
    def n_feat(self) -> int:
        return feature_count(self.kind, self.degree)

    @property
    def cheby_coeffs(self) -> torch.Tensor:
        """JOD [input, output, degree+1] view (tensor.py:26-28; original ChebyKAN layout)."""
        return self.coeff_doj.permute(2, 1, 0)

    @torch.no_grad()
    def reset_parameters(self, seed: int | None = None) -> None:
        s = 1.0 / math.sqrt(self.input_dim * self.n_feat)
        if seed is None:
            self.coeff_doj.uniform_(-s, s)
        else:
            rng = np.random.default_rng(seed)
            jod = rng.uniform(-s, s, size=self.input_dim * self.output_dim * self.n_feat)
            jod = jod.reshape(self.input_dim, self.output_dim, self.n_feat).transpose(2, 1, 0)
            self.coeff_doj.copy_(torch.from_numpy(np.ascontiguousarray(jod)).to(torch.float32))
        if self.bias is not None:
            self.bias.zero_()

    @torch.no_grad()
    def load_jod(self, c_jod) -> None:
        """Load coefficients given in JOD [I, O, K] order (reorder_to_doj, tensor.py:77-82)."""
        c = torch.as_tensor(c_jod, dtype=torch.float32)
        if tuple(c.shape) != (self.input_dim, self.output_dim, self.n_feat):
            raise ValueError(f"expected JOD shape {(self.input_dim, self.output_dim, self.n_feat)}, got {tuple(c.shape)}")
        self.coeff_doj.copy_(c.permute(2, 1, 0).contiguous())

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.shape[-1] != self.input_dim:
            raise ValueError(f"expected input shape (batch, {self.input_dim}), got {tuple(x.shape)}")
        lead = x.shape[:-1]
        want_cache = torch.is_grad_enabled() and self.coeff_doj.requires_grad
        y = ChebyKANFunction.apply(x.reshape(-1, self.input_dim), self.coeff_doj, self.bias, self._state, want_cache)
        return y.reshape(*lead, self.output_dim)

    def invalidate_prep(self) -> None:
        """Force the next forward to re-split the coefficients.  Needed after
        writes the autograd version counter does not see: ``coeff_doj.data``
        in-place ops (EMA, clipping), raw-pointer kernels, CUDA-graph replays
        of an optimizer step.  ``load_jod``, ``reset_parameters``, in-place ops
        on the parameter itself, the library's Adam and load_state_dict bump
        the counter and need nothing."""
        self._state.invalidate()

    def extra_repr(self) -> str:
        return (f"input_dim={self.input_dim}, output_dim={self.output_dim}, degree={self.degree}, "
                f"kind={self.kind.value}, basis_path={self.basis_path.value}, bias={self.bias is not None}, "
                f"lut_size={self.lut_size}")


# The layer is basis-generic; the reference calls it a KAN layer.
KANLayer = ChebyKANLayer
