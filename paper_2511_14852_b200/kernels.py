"""Operator API of the fused ChebyKAN layer (drop-in for polykan.kernels).

Reference: /root/reference/pkg/src/polykan/kernels.py.  ``fused_forward``
(kernels.py:351-371) and ``backward_fused`` (kernels.py:374-447) keep their
names, argument meaning and ValueError wording; the work runs in the sm_100a
kernels of libchebykan.so on the caller's current CUDA stream.  Tensors are
torch CUDA tensors (fp32 compute; inputs of other dtypes are converted like
the reference's ``np.asarray(x, dtype=float64)``).
"""
from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from enum import Enum

import torch

from . import _lib
from .basis import BasisKind, as_kind, degree_for
from .lut import ExactBasis, exact_basis
from .tensor import CoeffTensor, Layout


class BasisPath(Enum):
    LUT_INTERP = "lut"
    EXACT_RECURRENCE = "exact"


@dataclass(frozen=True)
class KernelMode:
    """Basis evaluation path and tanh chain-rule choice (kernels.py:35-44)."""

    basis_path: BasisPath = BasisPath.LUT_INTERP
    include_tanh_jacobian: bool = True


LUT_MODE = KernelMode(BasisPath.LUT_INTERP)
EXACT_MODE = KernelMode(BasisPath.EXACT_RECURRENCE)


@dataclass(frozen=True)
class TileSchedule:
    """Reference CPU tiling descriptor (kernels.py:51-105).

    Accepted for signature compatibility and validated the same way; the
    B200 kernels choose their own tensor-core tiling (128 x 256 MMA tiles),
    so the schedule does not change results.
    """

    tile_in: int
    tile_out: int
    lane_x: int
    lane_y: int
    g_x: int
    g_y: int
    d_in: int
    d_out: int

    def __post_init__(self) -> None:
        if min(self.tile_in, self.tile_out, self.lane_x, self.lane_y) < 1:
            raise ValueError("tile and lane sizes must be >= 1")
        if self.tile_out != self.lane_y:
            raise ValueError("output-aligned schedule requires tile_out == lane_y")
        if self.d_in < 1 or self.d_out < 1:
            raise ValueError("d_in and d_out must be >= 1")
        if self.g_x != math.ceil(self.d_in / self.tile_in):
            raise ValueError("g_x does not match ceil(d_in / tile_in)")
        if self.g_y != math.ceil(self.d_out / self.tile_out):
            raise ValueError("g_y does not match ceil(d_out / tile_out)")

    @classmethod
    def for_dims(cls, d_in: int, d_out: int, tile_in: int = 64, tile_out: int = 32, lane_x: int = 8,
                 lane_y: int | None = None) -> "TileSchedule":
        if d_in < 1 or d_out < 1:
            raise ValueError("d_in and d_out must be >= 1")
        lane_y = tile_out if lane_y is None else lane_y
        return cls(tile_in, tile_out, lane_x, lane_y, math.ceil(d_in / tile_in), math.ceil(d_out / tile_out),
                   d_in, d_out)


@dataclass
class PartialBuffer:
    """Partial-stage workspace (kernels.py:108-137) on the device; flat order
    gIdx = (tileO * g_x + tileI) * B * tile_out + b * tile_out + t_y.  Slots of
    padding lanes of a ragged last output tile stay zero; ``write_counts``
    (instrumented buffers) is incremented by the partial kernel itself on
    every store (atomically), so it shows one write per real slot."""

    g_x: int
    g_y: int
    batch: int
    tile_out: int
    data: torch.Tensor
    write_counts: torch.Tensor | None = None

    @classmethod
    def allocate(cls, sched: "TileSchedule", batch: int, instrument: bool = False, device=None) -> "PartialBuffer":
        if batch < 1:
            raise ValueError("batch must be >= 1")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        shape = (sched.g_y, sched.g_x, batch, sched.tile_out)
        return cls(sched.g_x, sched.g_y, batch, sched.tile_out, torch.zeros(shape, dtype=torch.float32, device=dev),
                   torch.zeros(shape, dtype=torch.int64, device=dev) if instrument else None)


@dataclass
class KernelCounters:
    """Merge/store counts (kernels.py:140-147).  The B200 kernels have no
    atomics either; the counts follow the reference's closed forms for the
    same logical reduction (one partial slot per input tile, one combine
    store per output, one ordered x-grad merge per output tile)."""

    forward_atomics: int = 0
    partial_writes: int = 0
    combine_stores: int = 0
    x_grad_merges: int = 0


@dataclass(frozen=True)
class AtomicCounts:
    fwd_baseline: int
    fwd_ours: int
    bwd_x_naive: int
    bwd_x_ours: int


def count_atomics(batch: int, d_in: int, d_out: int, sched: TileSchedule) -> AtomicCounts:
    """Closed-form atomic/merge counts of the reduction strategies (kernels.py:158-167)."""
    if min(batch, d_in, d_out) < 1:
        raise ValueError("batch, d_in, d_out must be >= 1")
    return AtomicCounts(batch * d_out * sched.g_x, 0, batch * d_in * d_out, batch * d_in * sched.g_y)


class NonFiniteInputError(ValueError):
    """Raised under validate=True; names the first offending element (kernels.py:170-183)."""

    def __init__(self, b: int, j: int):
        self.b = b
        self.j = j
        super().__init__(f"non-finite input at (b={b}, j={j})")


def _check_finite(x: torch.Tensor) -> None:
    bad = ~torch.isfinite(x)
    if bool(bad.any()):
        b, j = (int(v) for v in torch.nonzero(bad)[0].tolist())
        raise NonFiniteInputError(b, j)


class PreparedCoeff:
    """Tensor-core operands derived from fp32 DOJ coefficients.

    Holds the opaque prep buffer of ck_coeff_prepare: bf16 hi/lo split copies
    in DOJ and DJO order plus sum_i C[0,o,i].  Rebuild after every update of
    the coefficients (the Module does this by tracking the tensor version).
    """

    def __init__(self, coeff_doj: torch.Tensor):
        if coeff_doj.dim() != 3:
            raise ValueError("coefficients must be 3-D DOJ [K, O, I]")
        k, o, i = coeff_doj.shape
        self.n_feat, self.d_out, self.d_in = int(k), int(o), int(i)
        self.device = coeff_doj.device
        nbytes = _lib.lib().ck_coeff_prep_bytes(self.d_in, self.d_out, self.n_feat)
        self.buffer = torch.empty(nbytes, dtype=torch.uint8, device=coeff_doj.device)
        self.update(coeff_doj)

    def update(self, coeff_doj: torch.Tensor) -> None:
        c = coeff_doj.detach()
        if c.dtype != torch.float32 or not c.is_contiguous():
            c = c.to(torch.float32).contiguous()
        rc = _lib.lib().ck_coeff_prepare(c.data_ptr(), self.d_in, self.d_out, self.n_feat, self.buffer.data_ptr(),
                                         self.buffer.numel(), _lib.stream_handle(c.device))
        _lib.check(rc, "ck_coeff_prepare")
        self.key = self.key_of(coeff_doj)

    @staticmethod
    def key_of(coeff_doj: torch.Tensor) -> tuple:
        """Identity of the coefficient values the prep was built from: storage,
        address and autograd version counter (see _LayerState.prepared)."""
        return (coeff_doj.untyped_storage()._cdata, coeff_doj.data_ptr(), coeff_doj._version)

    def check(self) -> None:
        """Synchronous validation of the prep buffer's host record and device
        header against this layer shape (ck_coeff_prep_check)."""
        _lib.check(_lib.lib().ck_coeff_prep_check(self.buffer.data_ptr(), self.buffer.numel(), self.d_in, self.d_out,
                                                  self.n_feat), "ck_coeff_prep_check")


@contextlib.contextmanager
def chunk_rows(rows: int):
    """Temporarily set the rows per internal batch chunk of ck_forward /
    ck_backward (ck_set_chunk_rows; default 32768).  dC accumulates over the
    chunks in ascending order, so a small value runs a wide layer's
    multi-chunk accumulation on a small batch.  Process-wide: keep a forward
    and the backward that reuses its basis cache inside the same setting."""
    lib = _lib.lib()
    prev = lib.ck_set_chunk_rows(int(rows))
    try:
        yield
    finally:
        lib.ck_set_chunk_rows(prev)


def _as_f32(t: torch.Tensor, device) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    return t.to(device=device, dtype=torch.float32).contiguous()


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def basis_cache_bytes(batch: int, d_in: int, d_out: int, n_feat: int) -> int:
    """Bytes of the forward->backward basis cache (bf16 hi/lo planes, k >= 1);
    0 when the layer does not use basis planes (skinny d_out)."""
    return int(_lib.lib().ck_basis_cache_bytes(batch, d_in, d_out, n_feat))


def forward_raw(x: torch.Tensor, prep: PreparedCoeff, lut, bias: torch.Tensor | None,
                cache: torch.Tensor | None = None) -> torch.Tensor:
    """y = fused layer forward on prepared coefficients (x fp32 contiguous [B, I]).

    ``cache`` (uint8, >= basis_cache_bytes): keep the expanded basis for the
    backward of the same x.
    """
    b = x.shape[0]
    y = torch.empty((b, prep.d_out), dtype=torch.float32, device=x.device)
    lb = _lib.lib()
    ws = _workspace(lb.ck_forward_workspace_bytes(b, prep.d_in, prep.d_out, prep.n_feat), x.device)
    rc = lb.ck_forward(x.data_ptr(), b, prep.d_in, prep.d_out, lut.handle, prep.buffer.data_ptr(), prep.buffer.numel(),
                       _lib.ptr(bias),
                       y.data_ptr(), ws.data_ptr(), ws.numel(), _lib.ptr(cache), 0 if cache is None else cache.numel(),
                       _lib.stream_handle(x.device))
    _lib.check(rc, "ck_forward")
    return y


def backward_raw(x: torch.Tensor, dy: torch.Tensor, prep: PreparedCoeff, lut, jacobian: bool,
                 want_dx: bool = True, want_dc: bool = True, want_db: bool = True,
                 cache: torch.Tensor | None = None, dc_out: torch.Tensor | None = None,
                 db_out: torch.Tensor | None = None, grads_ready=None):
    """(dC DOJ, dX, db) on prepared coefficients; unrequested outputs are None.

    ``cache``: the basis cache filled by forward_raw on the same x (optional).
    ``dc_out`` / ``db_out``: contiguous fp32 tensors to write dC / db into
    (e.g. views of a data-parallel exchange buffer) instead of new ones.
    ``grads_ready``: a torch.cuda.Event recorded as soon as dC and db are
    final, before the last input-gradient GEMM (ck_backward's event).
    """
    b = x.shape[0]
    dev = x.device
    dx = torch.empty((b, prep.d_in), dtype=torch.float32, device=dev) if want_dx else None
    dc, db = None, None
    if want_dc:
        dc = dc_out if dc_out is not None else torch.empty((prep.n_feat, prep.d_out, prep.d_in), dtype=torch.float32,
                                                           device=dev)
        if tuple(dc.shape) != (prep.n_feat, prep.d_out, prep.d_in) or not dc.is_contiguous():
            raise ValueError("dc_out must be a contiguous [K, O, I] tensor")
    if want_db:
        db = db_out if db_out is not None else torch.empty((prep.d_out,), dtype=torch.float32, device=dev)
        if tuple(db.shape) != (prep.d_out,) or not db.is_contiguous():
            raise ValueError("db_out must be a contiguous [O] tensor")
    ev = None
    if grads_ready is not None:
        ev = grads_ready.cuda_event
        if not ev:  # torch creates the event lazily
            grads_ready.record()
            ev = grads_ready.cuda_event
    lb = _lib.lib()
    ws = _workspace(lb.ck_backward_workspace_bytes(b, prep.d_in, prep.d_out, prep.n_feat), dev)
    rc = lb.ck_backward(x.data_ptr(), dy.data_ptr(), b, prep.d_in, prep.d_out, lut.handle, prep.buffer.data_ptr(),
                        prep.buffer.numel(), 1 if jacobian else 0, _lib.ptr(dx), _lib.ptr(dc), _lib.ptr(db), ws.data_ptr(), ws.numel(),
                        _lib.ptr(cache), 0 if cache is None else cache.numel(), ev, _lib.stream_handle(dev))
    _lib.check(rc, "ck_backward")
    return dc, dx, db


def _resolve_kind(lut, kind) -> BasisKind:
    """kernels.py:186-191."""
    if lut is not None:
        return lut.kind
    if kind is not None:
        return as_kind(kind)
    raise ValueError("exact mode without a LUT requires an explicit basis kind")


def _basis_for(coeff: CoeffTensor, lut, sched: TileSchedule | None, mode: KernelMode, kind, what: str, device):
    """Validate like the reference and return the device basis handle:
    the LutTable (LUT mode) or the exact-evaluation handle (kernels.py:194-224)."""
    if coeff.layout is not Layout.DOJ:
        raise ValueError(f"{what} requires DOJ coefficient layout")
    if sched is not None and (sched.d_in != coeff.d_in or sched.d_out != coeff.d_out):
        raise ValueError("schedule dimensions do not match the coefficient tensor")
    if mode.basis_path is BasisPath.LUT_INTERP:
        if lut is None:
            raise ValueError("LUT mode requires a LutTable")
        if lut.n_features != coeff.n_feat:
            raise ValueError(f"LUT has {lut.n_features} features, coefficients expect {coeff.n_feat}")
        return lut
    bkind = _resolve_kind(lut, kind)
    dev = lut.device if lut is not None else device
    return exact_basis(bkind, degree_for(bkind, coeff.n_feat), device=dev)


def _device_for(x, lut) -> torch.device:
    if lut is not None:
        return torch.device("cuda", lut.device)
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return torch.device("cuda", torch.cuda.current_device())


def fused_forward(x, coeff: CoeffTensor, lut, sched: TileSchedule | None = None, mode: KernelMode = LUT_MODE,
                  bias=None, *, workers: int = 1, counters: KernelCounters | None = None, validate: bool = False,
                  kind: BasisKind | None = None) -> torch.Tensor:
    """y[b,o] = sum_j sum_k C[k,o,j] B_k(tanh x[b,j]) + bias[o]; returns (B, d_out) fp32.

    kernels.py:351-371 (forward_partial 263-290 + combine 321-348).  ``workers``
    is accepted for signature compatibility (the GPU kernels own the
    parallelism).
    """
    dev = _device_for(x, lut)
    basis = _basis_for(coeff, lut, sched, mode, kind, "forward_partial", dev)
    x = _as_f32(x, dev)
    if x.dim() != 2:
        raise ValueError(f"input must be 2-D (batch, d_in), got shape {tuple(x.shape)}")
    if x.shape[1] != coeff.d_in:
        raise ValueError(f"input width {x.shape[1]} != coefficient d_in {coeff.d_in}")
    if bias is not None:
        bias = _as_f32(bias, dev)
        if tuple(bias.shape) != (coeff.d_out,):
            raise ValueError(f"bias must have shape ({coeff.d_out},), got {tuple(bias.shape)}")
    if validate:
        _check_finite(x)
    prep = PreparedCoeff(_as_f32(coeff.as3d(), dev))
    y = forward_raw(x, prep, basis, bias)
    if counters is not None:
        sched = sched or TileSchedule.for_dims(coeff.d_in, coeff.d_out)
        counters.partial_writes += x.shape[0] * coeff.d_out * sched.g_x
        counters.combine_stores += x.shape[0] * coeff.d_out
    return y


def backward_fused(x, coeff: CoeffTensor, dy, lut, sched: TileSchedule | None = None, mode: KernelMode = LUT_MODE,
                   *, workers: int = 1, counters: KernelCounters | None = None, validate: bool = False,
                   kind: BasisKind | None = None):
    """(coeff_grad DOJ CoeffTensor, x_grad (B, d_in)); kernels.py:374-447."""
    dev = _device_for(x, lut)
    basis = _basis_for(coeff, lut, sched, mode, kind, "backward_fused", dev)
    x = _as_f32(x, dev)
    dy = _as_f32(dy, dev)
    if x.dim() != 2 or dy.dim() != 2:
        raise ValueError("x and dy must be 2-D")
    if x.shape[1] != coeff.d_in:
        raise ValueError(f"input width {x.shape[1]} != coefficient d_in {coeff.d_in}")
    if tuple(dy.shape) != (x.shape[0], coeff.d_out):
        raise ValueError(f"dy must have shape ({x.shape[0]}, {coeff.d_out}), got {tuple(dy.shape)}")
    if validate:
        _check_finite(x)
        _check_finite(dy)
    prep = PreparedCoeff(_as_f32(coeff.as3d(), dev))
    dc, dx, _ = backward_raw(x, dy, prep, basis, mode.include_tanh_jacobian, want_db=False)
    if counters is not None:
        sched = sched or TileSchedule.for_dims(coeff.d_in, coeff.d_out)
        counters.x_grad_merges += x.shape[0] * coeff.d_in * sched.g_y
    return CoeffTensor(coeff.d_in, coeff.d_out, coeff.degree, Layout.DOJ, dc), dx


def forward_partial(x, coeff: CoeffTensor, lut, sched: TileSchedule, mode: KernelMode, out: PartialBuffer, *,
                    workers: int = 1, counters: KernelCounters | None = None, validate: bool = False,
                    kind: BasisKind | None = None) -> None:
    """Partial stage (kernels.py:263-318): slot (tileO, tileI, b, t_y) receives
    sum_{j in tile} sum_k coeff[k, out, j] B_k(tanh x[b, j]); each slot has one
    writer.  Runs on the GPU (ck_forward_partial, fp32 CUDA cores); the fused
    tensor-core path is fused_forward."""
    dev = out.data.device
    basis = _basis_for(coeff, lut, None, mode, kind, "forward_partial", dev)
    x = _as_f32(x, dev)
    if x.dim() != 2:
        raise ValueError(f"input must be 2-D (batch, d_in), got shape {tuple(x.shape)}")
    if x.shape[1] != coeff.d_in:
        raise ValueError(f"input width {x.shape[1]} != coefficient d_in {coeff.d_in}")
    if sched.d_in != coeff.d_in or sched.d_out != coeff.d_out:
        raise ValueError("schedule dimensions do not match the coefficient tensor")
    if (out.g_x, out.g_y, out.batch, out.tile_out) != (sched.g_x, sched.g_y, x.shape[0], sched.tile_out):
        raise ValueError("partial buffer does not match the schedule and batch")
    if validate:
        _check_finite(x)
    c = _as_f32(coeff.as3d(), dev)
    rc = _lib.lib().ck_forward_partial(x.data_ptr(), x.shape[0], coeff.d_in, coeff.d_out, basis.handle, c.data_ptr(),
                                       sched.tile_in, sched.tile_out, out.data.data_ptr(), _lib.ptr(out.write_counts),
                                       _lib.stream_handle(dev))
    _lib.check(rc, "ck_forward_partial")
    if counters is not None:
        counters.partial_writes += x.shape[0] * sched.d_out * sched.g_x


def combine(partial: PartialBuffer, sched: TileSchedule, bias=None, *,
            counters: KernelCounters | None = None) -> torch.Tensor:
    """Combine stage (kernels.py:321-348): fold input tiles in ascending order,
    add the bias; one store per output (ck_combine)."""
    dev = partial.data.device
    if bias is not None:
        bias = _as_f32(bias, dev)
        if tuple(bias.shape) != (sched.d_out,):
            raise ValueError(f"bias must have shape ({sched.d_out},), got {tuple(bias.shape)}")
    y = torch.empty((partial.batch, sched.d_out), dtype=torch.float32, device=dev)
    rc = _lib.lib().ck_combine(partial.data.data_ptr(), partial.batch, sched.d_out, partial.g_x, partial.tile_out,
                               _lib.ptr(bias), y.data_ptr(), _lib.stream_handle(dev))
    _lib.check(rc, "ck_combine")
    if counters is not None:
        counters.combine_stores += partial.batch * sched.d_out
    return y


def _exact_for(kind, n_feat: int, trig: bool, device) -> ExactBasis:
    bkind = as_kind(kind) if kind is not None else BasisKind.CHEBYSHEV
    if trig and bkind is not BasisKind.CHEBYSHEV:
        raise ValueError("the trig path applies to the Chebyshev basis only")
    return exact_basis(bkind, degree_for(bkind, n_feat), device=device, trig=trig)


def reference_forward(x, coeff: CoeffTensor, degree: int, *, trig: bool = False,
                      kind: BasisKind | None = None) -> torch.Tensor:
    """Exact (table-free) evaluation, kernels.py:450-478: basis_rows (or
    cos(n arccos t) with ``trig``) at tanh(x), contracted with JOD coefficients.
    Runs on the B200 kernels with an exact-evaluation handle."""
    if coeff.layout is not Layout.JOD:
        raise ValueError("reference_forward expects JOD coefficient layout")
    if degree != coeff.degree:
        raise ValueError(f"degree {degree} does not match coefficients ({coeff.degree})")
    dev = _device_for(x, None)
    x = _as_f32(x, dev)
    if x.dim() != 2 or x.shape[1] != coeff.d_in:
        raise ValueError(f"input must be (batch, {coeff.d_in}), got {tuple(x.shape)}")
    basis = _exact_for(kind, coeff.n_feat, trig, dev)
    prep = PreparedCoeff(_as_f32(coeff.as3d().permute(2, 1, 0), dev))
    return forward_raw(x, prep, basis, None)


def reference_backward(x, coeff: CoeffTensor, dy, *, trig: bool = False, kind: BasisKind | None = None,
                       include_tanh_jacobian: bool = True):
    """Exact backward with analytic derivatives, kernels.py:481-510; returns
    (JOD coefficient gradient, x_grad)."""
    if coeff.layout is not Layout.JOD:
        raise ValueError("reference_backward expects JOD coefficient layout")
    dev = _device_for(x, None)
    x = _as_f32(x, dev)
    dy = _as_f32(dy, dev)
    basis = _exact_for(kind, coeff.n_feat, trig, dev)
    prep = PreparedCoeff(_as_f32(coeff.as3d().permute(2, 1, 0), dev))
    dc, dx, _ = backward_raw(x, dy, prep, basis, include_tanh_jacobian, want_db=False)
    return CoeffTensor(coeff.d_in, coeff.d_out, coeff.degree, Layout.JOD, dc.permute(2, 1, 0).contiguous()), dx


def count_flops(batch: int, d_in: int, d_out: int, degree: int, n_feat: int | None = None) -> dict:
    """Algorithmic FLOPs of one layer call; K = n_feat
    (degree + 1 unless given, e.g. 2*degree + 1 for Fourier)."""
    k = degree + 1 if n_feat is None else n_feat
    fwd = 2 * batch * d_in * d_out * k
    bwd = 2 * batch * d_in * d_out * k + 2 * batch * d_in * d_out * (k - 1)
    return {"fwd": fwd, "bwd": bwd, "train": fwd + bwd}
