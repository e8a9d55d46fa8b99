"""Data-parallel training of ChebyKAN layers: batch sharded, dC/db allreduced.

One process per GPU (torchrun), ``torch.distributed`` with NCCL over
NVLink/NVSwitch.  The forward and the input gradient are row-independent,
so the only exchange per step is one allreduce(sum) of the concatenated
fp32 coefficient and bias gradients of every ChebyKAN layer (SURVEY.md
section 8(e)).  Rank shards are contiguous row blocks of the global batch.
"""
from __future__ import annotations

import ctypes

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


class GradientAllreducer:
    """Flatten -> one allreduce -> scatter back, for a fixed parameter list.

    The flat buffer is allocated once; per step the gradients are packed in a
    fixed order, reduced with a single collective (sum, or mean when
    ``average``), and copied back.  With NCCL the reduction order is fixed
    for a given world size, so results are run-to-run reproducible.
    """

    def __init__(self, params: list[torch.nn.Parameter], group=None, average: bool = False):
        self.params = list(params)
        self.group = group
        self.average = average
        n = sum(p.numel() for p in self.params)
        dev = self.params[0].device if self.params else torch.device("cpu")
        self.flat = torch.empty(n, dtype=torch.float32, device=dev)

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4

    def __call__(self) -> None:
        if not dist.is_available() or not dist.is_initialized():
            return
        world = dist.get_world_size(self.group)
        if world == 1:
            return
        off = 0
        views = []
        for p in self.params:
            n = p.numel()
            v = self.flat[off:off + n]
            if p.grad is None:
                v.zero_()
            else:
                v.copy_(p.grad.reshape(-1))
            views.append((p, v))
            off += n
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        if self.average:
            self.flat.div_(world)
        for p, v in views:
            if p.grad is None:
                p.grad = v.view_as(p).clone()
            else:
                p.grad.copy_(v.view_as(p))


class PeerAllreducer(GradientAllreducer):
    """Deterministic allreduce of the flat gradient over peer memory.

    Same packing as GradientAllreducer, but the exchange is the library's own
    kernel (ck_allreduce_peers): every rank maps every peer's flat buffer via
    CUDA IPC (NVLink/NVSwitch peers, or processes sharing a device); rank r
    sums shard r over ranks 0..R-1 in ascending order and stores it into every
    rank's buffer.  Results are bit-identical on all ranks and across runs
    without relying on NCCL's algorithm choice.  The process group (any
    backend) only carries the handle exchange and the two barriers around the
    kernel.  Up to 8 ranks.
    """

    def __init__(self, params: list[torch.nn.Parameter], group=None, average: bool = False):
        super().__init__(params, group, average)
        self._peers = None
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            self._open()

    def _open(self) -> None:
        lib = _lib.lib()
        world = dist.get_world_size(self.group)
        if world > 8:
            raise ValueError("PeerAllreducer supports up to 8 ranks")
        handle = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64()
        _lib.check(lib.ck_ipc_handle(self.flat.data_ptr(), handle, ctypes.byref(off)), "ck_ipc_handle")
        mine = (bytes(handle), off.value)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=self.group)
        me = dist.get_rank(self.group)
        ptrs = []
        opened = []
        err = None
        for r, (h, o) in enumerate(allh):
            if r == me:
                ptrs.append(self.flat.data_ptr())
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * 64).from_buffer_copy(h)
            rc = lib.ck_ipc_open(buf, o, ctypes.byref(p))
            if rc != 0:
                err = _lib.last_error() or f"code {rc}"
                break
            opened.append((p.value, o))
            ptrs.append(p.value)
        # every rank must have mapped every peer before any uses the mappings:
        # agree on it, so a rank-local failure sends all ranks to the fallback
        # together instead of leaving the others in the self-test's barriers
        dev = self.flat.device
        on = dev if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        ok = torch.tensor([0.0 if err else 1.0], device=on)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if ok.item() != 1.0:
            for ptr, o in opened:
                lib.ck_ipc_close(ctypes.c_void_p(ptr), o)
            raise ValueError(f"peer-memory mapping failed on some rank ({err or 'a peer'})")
        self._offsets = [o for _, o in allh]
        self._peers = (ctypes.c_void_p * world)(*ptrs)
        self._rank, self._world = me, world
        self._self_test()

    def _self_test(self) -> None:
        """One exchange on a known pattern before use: every rank must see
        sum_r (r + 1) everywhere, agreed by all ranks, else ValueError (the
        caller falls back to NCCL)."""
        dev = self.flat.device
        saved = self.flat.clone()
        self.flat.fill_(float(self._rank + 1))
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)
        _lib.check(_lib.lib().ck_allreduce_peers(self._peers, self._world, self._rank, self.flat.numel(),
                                                 _lib.stream_handle(dev)), "ck_allreduce_peers")
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)
        want = self._world * (self._world + 1) / 2
        on = dev if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        ok = torch.tensor([1.0 if bool((self.flat == want).all()) else 0.0], device=on)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        self.flat.copy_(saved)
        if ok.item() != 1.0:
            self.close()
            raise ValueError("peer-memory allreduce self-test failed")

    def __call__(self) -> None:
        if self._peers is None:
            return
        views = []
        off = 0
        for p in self.params:
            n = p.numel()
            v = self.flat[off:off + n]
            if p.grad is None:
                v.zero_()
            else:
                v.copy_(p.grad.reshape(-1))
            views.append((p, v))
            off += n
        dev = self.flat.device
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)  # every rank's gradient is in its buffer
        _lib.check(_lib.lib().ck_allreduce_peers(self._peers, self._world, self._rank, self.flat.numel(),
                                                 _lib.stream_handle(dev)), "ck_allreduce_peers")
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)  # every shard has been written everywhere
        if self.average:
            self.flat.div_(self._world)
        for p, v in views:
            if p.grad is None:
                p.grad = v.view_as(p).clone()
            else:
                p.grad.copy_(v.view_as(p))

    def close(self) -> None:
        if self._peers is None:
            return
        lib = _lib.lib()
        for r in range(self._world):
            if r != self._rank:
                lib.ck_ipc_close(ctypes.c_void_p(self._peers[r]), self._offsets[r])
        self._peers = None


def allreduce_gradients(module: nn.Module, group=None, average: bool = False) -> None:
    """One-shot helper: allreduce every ChebyKAN gradient of ``module``."""
    GradientAllreducer(chebykan_parameters(module), group, average)()
