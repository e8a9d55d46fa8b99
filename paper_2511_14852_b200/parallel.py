"""Data-parallel training of ChebyKAN layers: batch sharded, dC/db exchanged.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.  The
forward and the input gradient are row-independent, so the only exchange per
step is the sum over ranks of every ChebyKAN layer's fp32 coefficient and
bias gradients.  Rank shards are contiguous row
blocks of the global batch.

Two reducers share one layout -- a flat fp32 buffer holding every layer's
[dC, db] at 16-byte aligned offsets:

* ``GradientAllreducer``: one NCCL ``all_reduce(SUM)`` of the flat buffer
  (NCCL_ALGO=Ring / NCCL_PROTO=Simple pinned for a fixed reduction order).
* ``PeerAllreducer``: the library's own fixed-order reduce over CUDA-IPC
  peer memory (ck_allreduce_peers_flags), synchronised by device-side flags
  in the mapped buffers -- no host synchronize, no host barrier.

``bind(module)`` makes the backward kernels write dC and db straight into
the flat buffer (no pack / unpack copies: the parameters' ``.grad`` become
views of it) and, for the peer reducer, enqueues each layer's exchange on a
side stream as soon as ck_backward's grads-ready event fires -- before the
layer's last input-gradient GEMM, and while the earlier layers' backward
runs.  The persistent GEMMs then leave a few SMs free for the exchange
kernel (ck_set_gemm_sm_reserve).
"""
from __future__ import annotations

import contextlib
import ctypes
import os
import weakref

import torch
import torch.distributed as dist
from torch import nn

from . import _lib
from .layer import ChebyKANLayer


def shard_bounds(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) rows of rank's shard; earlier ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    base, rem = divmod(global_batch, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def chebykan_parameters(module: nn.Module) -> list[torch.nn.Parameter]:
    """Gradient-carrying parameters in a fixed order (module traversal order)."""
    params: list[torch.nn.Parameter] = []
    for m in module.modules():
        if isinstance(m, ChebyKANLayer):
            params.append(m.coeff_doj)
            if m.bias is not None:
                params.append(m.bias)
    return params


def deterministic_nccl_env() -> None:
    """Pin NCCL to one algorithm and protocol (a fixed reduction order, so
    the summed gradients are bit-reproducible run to run at a fixed world
    size).  NCCL reads these when a communicator is created: call before the
    first collective (GradientAllreducer's constructor does, and warns when
    the process group already has an explicit other choice)."""
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")


def _align4(n: int) -> int:
    return (n + 3) // 4 * 4


class _Layout:
    """16-byte aligned slots of every parameter in one flat fp32 buffer."""

    def __init__(self, params):
        self.params = list(params)
        self.offsets = []
        off = 0
        for p in self.params:
            self.offsets.append(off)
            off += _align4(p.numel())
        self.n = off

    def view(self, flat, i):
        p = self.params[i]
        return flat[self.offsets[i]:self.offsets[i] + p.numel()].view_as(p)


class GradientAllreducer:
    """Sum (or mean) of the parameters' gradients over the process group.

    The flat buffer is allocated once.  Unbound, each call packs the
    gradients into it, runs one all_reduce and copies them back; after
    ``bind(module)`` the backward writes the gradients into the buffer
    directly and the call is one all_reduce in place.
    """

    def __init__(self, params: list[torch.nn.Parameter], group=None, average: bool = False, extra_floats: int = 0):
        deterministic_nccl_env()
        self.group = group
        self.average = average
        self.layout = _Layout(params)
        self.params = self.layout.params
        dev = self.params[0].device if self.params else torch.device("cpu")
        self._storage = torch.zeros(self.layout.n + extra_floats, dtype=torch.float32, device=dev)
        self.flat = self._storage[:self.layout.n]
        self.views = [self.layout.view(self.flat, i) for i in range(len(self.params))]
        self._sinks: list = []
        self._no_sync = False

    @property
    def nbytes(self) -> int:
        return self.layout.n * 4

    def _world(self) -> int:
        if not dist.is_available() or not dist.is_initialized():
            return 1
        return dist.get_world_size(self.group)

    # --- in-place gradients -------------------------------------------------
    def bind(self, module: nn.Module) -> "GradientAllreducer":
        """Have every ChebyKAN layer of ``module`` write its dC / db into the
        flat buffer (the module's ChebyKAN parameters must be this reducer's
        parameters, in chebykan_parameters order)."""
        by_param = {id(p): i for i, p in enumerate(self.params)}
        for m in module.modules():
            if not isinstance(m, ChebyKANLayer):
                continue
            ic = by_param.get(id(m.coeff_doj))
            ib = by_param.get(id(m.bias)) if m.bias is not None else None
            if ic is None or (m.bias is not None and ib is None):
                raise ValueError("bind: the module's parameters are not this reducer's")
            sink = _GradSink(self, m, ic, ib)
            m._state.grad_sink = sink
            self._sinks.append(sink)
        return self

    @contextlib.contextmanager
    def no_sync(self):
        """Backward passes inside accumulate gradients without starting an
        exchange (micro-batches before the last one of a step)."""
        prev, self._no_sync = self._no_sync, True
        try:
            yield
        finally:
            self._no_sync = prev

    def _pack(self) -> list:
        """Copy gradients that are not already the buffer's views into it."""
        copied = []
        for p, v in zip(self.params, self.views):
            if p.grad is None:
                v.zero_()
            elif p.grad.data_ptr() != v.data_ptr():
                v.copy_(p.grad.reshape(v.shape))
                copied.append((p, v))
            # else: the backward wrote it in place
        return copied

    def _unpack(self, copied) -> None:
        for p, v in zip(self.params, self.views):
            if p.grad is None:
                p.grad = v  # (a parameter without a local gradient: the sum of the others')
        for p, v in copied:
            p.grad.copy_(v)

    def __call__(self) -> None:
        world = self._world()
        if world == 1:
            for s in self._sinks:
                s.reset()
            return
        copied = self._pack()
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        if self.average:
            self.flat.div_(world)
        self._unpack(copied)
        for s in self._sinks:
            s.reset()


# Per-process reference-counted IPC mappings: several reducers (or buffers
# sharing one caching-allocator segment) map a peer's segment once, and it is
# unmapped only when the last user closes it.
_IPC_MAPS: dict = {}


def _ipc_open(handle: bytes, offset: int) -> int:
    lib = _lib.lib()
    ent = _IPC_MAPS.get(handle)
    if ent is None:
        p = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        _lib.check(lib.ck_ipc_open(buf, 0, ctypes.byref(p)), "ck_ipc_open")
        ent = _IPC_MAPS[handle] = [p.value, 0]
    ent[1] += 1
    return ent[0] + offset


def _ipc_close(handle: bytes) -> None:
    ent = _IPC_MAPS.get(handle)
    if ent is None:
        return
    ent[1] -= 1
    if ent[1] == 0:
        del _IPC_MAPS[handle]
        _lib.lib().ck_ipc_close(ctypes.c_void_p(ent[0]), 0)


class PeerAllreducer(GradientAllreducer):
    """Deterministic sum of the flat gradient buffer over peer memory.

    Every rank maps every peer's buffer (plus its flag words) via CUDA IPC
    (NVLink / NVSwitch peers, or processes sharing a device).  Rank r sums
    shard r over ranks 0..R-1 in ascending order and stores it into every
    rank's buffer, so all ranks hold bit-identical gradients, run to run,
    independent of NCCL's algorithm choice.  The exchange kernel
    synchronises with the other ranks through flags in the mapped memory;
    the process group (any backend) only carries the one-time handle
    exchange.  Up to 8 ranks.

    ``overlap_sms``: SMs the GEMMs leave free while a bound module's backward
    runs (the exchange kernels of finished layers run there concurrently).
    """

    def __init__(self, params: list[torch.nn.Parameter], group=None, average: bool = False, overlap_sms: int = 4):
        words = int(_lib.lib().ck_peer_flag_words())
        super().__init__(params, group, average, extra_floats=2 * words + 4)
        base = self._storage.data_ptr() + 4 * self.layout.n
        base = (base + 7) // 8 * 8
        self._flag_off = base - self._storage.data_ptr()  # bytes
        self._peers = None
        self._epoch = 0
        self.overlap_sms = int(overlap_sms)
        self._side = None
        if self._world() > 1:
            self._open()

    def _open(self) -> None:
        lib = _lib.lib()
        world = dist.get_world_size(self.group)
        if world > 8:
            raise ValueError("PeerAllreducer supports up to 8 ranks")
        handle = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64()
        _lib.check(lib.ck_ipc_handle(self._storage.data_ptr(), handle, ctypes.byref(off)), "ck_ipc_handle")
        mine = (bytes(handle), off.value)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=self.group)
        me = dist.get_rank(self.group)
        bases, opened, err = [], [], None
        for r, (h, o) in enumerate(allh):
            if r == me:
                bases.append(self._storage.data_ptr())
                continue
            try:
                bases.append(_ipc_open(h, o))
                opened.append(h)
            except Exception as exc:  # noqa: BLE001 (agreed on below)
                err = str(exc)
                break
        # every rank must have mapped every peer before any uses the mappings:
        # agree on it, so a rank-local failure sends all ranks to the fallback
        on = self.flat.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        ok = torch.tensor([0.0 if err else 1.0], device=on)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if ok.item() != 1.0:
            for h in opened:
                _ipc_close(h)
            raise ValueError(f"peer-memory mapping failed on some rank ({err or 'a peer'})")
        self._handles = opened
        self._peers = (ctypes.c_void_p * world)(*bases)
        self._flags = (ctypes.c_void_p * world)(*[b + self._flag_off for b in bases])
        self._rank, self._world_n = me, world
        self._side = torch.cuda.Stream(device=self.flat.device)
        self._self_test()

    def _exchange(self, lo: int, n: int, stream, max_blocks: int = 0) -> None:
        self._epoch += 1
        _lib.check(_lib.lib().ck_allreduce_peers_flags(self._peers, self._flags, self._world_n, self._rank, lo, n,
                                                        self._epoch, max_blocks, stream.cuda_stream),
                   "ck_allreduce_peers_flags")

    def _self_test(self) -> None:
        """One exchange on a known pattern before use: every rank must see
        sum_r (r + 1) everywhere, agreed by all ranks, else ValueError (the
        caller falls back to NCCL)."""
        dev = self.flat.device
        saved = self.flat.clone()
        self.flat.fill_(float(self._rank + 1))
        self._exchange(0, self.layout.n, torch.cuda.current_stream(dev))
        torch.cuda.current_stream(dev).synchronize()
        want = self._world_n * (self._world_n + 1) / 2
        on = dev if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        ok = torch.tensor([1.0 if bool((self.flat == want).all()) else 0.0], device=on)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        self.flat.copy_(saved)
        if ok.item() != 1.0:
            self.close()
            raise ValueError("peer-memory allreduce self-test failed")

    # called by _GradSink from a layer's backward
    def _launch_layer(self, sink: "_GradSink") -> None:
        self._side.wait_event(sink.event)
        lo = self.layout.offsets[sink.ic]
        hi = self.layout.offsets[sink.ib] + self.params[sink.ib].numel() if sink.ib is not None else \
            lo + self.params[sink.ic].numel()
        self._exchange(lo, _align4(hi - lo), self._side, max_blocks=2 * max(1, self.overlap_sms))
        # (the parameters' .grad -- views of the buffer -- are read on the
        # default stream only after __call__ joins the side stream)

    def _begin_backward(self) -> None:
        if self.overlap_sms > 0:
            _lib.lib().ck_set_gemm_sm_reserve(self.overlap_sms)

    def __call__(self) -> None:
        if self._peers is None:
            for s in self._sinks:
                s.reset()
            return
        cur = torch.cuda.current_stream(self.flat.device)
        _lib.lib().ck_set_gemm_sm_reserve(0)
        # slots of layers whose exchange already ran on the side stream
        inplace = set()
        for s in self._sinks:
            if s.launched:
                inplace.update(i for i in (s.ic, s.ib) if i is not None)
        pending = [i for i in range(len(self.params)) if i not in inplace]
        copied = []
        for i in pending:
            p, v = self.params[i], self.views[i]
            if p.grad is None:
                v.zero_()
            elif p.grad.data_ptr() != v.data_ptr():
                v.copy_(p.grad.reshape(v.shape))
                copied.append((p, v))
        if len(pending) == len(self.params):
            self._exchange(0, self.layout.n, cur)  # nothing bound: one exchange of the whole buffer
        else:
            for i in pending:
                self._exchange(self.layout.offsets[i], _align4(self.params[i].numel()), cur)
        cur.wait_stream(self._side)
        if self.average:
            self.flat.div_(self._world_n)
        for i in inplace:
            self.params[i].grad = self.views[i]  # (also when autograd copied instead of taking the view)
        self._unpack(copied)
        for s in self._sinks:
            s.reset()

    def close(self) -> None:
        if self._peers is None:
            return
        for h in self._handles:
            _ipc_close(h)
        self._peers = None


class _GradSink:
    """A bound layer's side of the reducer: its slots in the flat buffer, the
    grads-ready event ck_backward records, and the per-step state."""

    def __init__(self, reducer: GradientAllreducer, layer: ChebyKANLayer, ic: int, ib):
        self._reducer = weakref.ref(reducer)
        self._layer = weakref.ref(layer)
        self.ic, self.ib = ic, ib
        self.event = torch.cuda.Event()
        self.launched = False

    def try_begin(self):
        """(dc_out, db_out, event) when this step's gradients can go to the
        buffer in place -- none accumulated yet -- else None."""
        red, layer = self._reducer(), self._layer()
        if red is None or layer is None or self.launched:
            return None
        if layer.coeff_doj.grad is not None or (layer.bias is not None and layer.bias.grad is not None):
            return None  # accumulating over micro-batches: autograd adds to the existing .grad
        if isinstance(red, PeerAllreducer) and red._peers is not None and not red._no_sync:
            red._begin_backward()
        db = red.views[self.ib] if self.ib is not None else None
        return red.views[self.ic], db, self.event

    def done(self) -> None:
        red = self._reducer()
        if red is None or red._no_sync:
            return  # in place, but more micro-batches will add to it: exchanged at the step's call
        self.launched = True
        if isinstance(red, PeerAllreducer) and red._peers is not None:
            red._launch_layer(self)

    def reset(self) -> None:
        self.launched = False


def allreduce_gradients(module: nn.Module, group=None, average: bool = False) -> None:
    """One-shot helper: allreduce every ChebyKAN gradient of ``module``."""
    GradientAllreducer(chebykan_parameters(module), group, average)()
