"""Device optimizer: Adam with bias correction on the library's own kernel.

The update rule is the reference trainer's ``adam_step`` (model.py:247-266):
m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2, p -= lr * m_hat / (sqrt(v_hat) + eps),
one step counter per optimizer, an optional per-step ``lr_scale`` (the cosine
decay of network_train, model.py:447-451).  ``ck_adam_step`` runs it in place
on one fp32 tensor (one HBM pass over p, g, m, v); ``Adam.step`` updates all
of a device's parameters with one ``ck_adam_step_multi`` launch.
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib


def adam_update(param: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, lr: float,
                beta1: float, beta2: float, eps: float, step: int) -> None:
    """One in-place Adam update of a contiguous fp32 CUDA tensor (ck_adam_step)."""
    for t in (param, grad, m, v):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("adam_update expects contiguous float32 CUDA tensors")
    if not (param.numel() == grad.numel() == m.numel() == v.numel()):
        raise ValueError("parameter, gradient and moment sizes differ")
    rc = _lib.lib().ck_adam_step(param.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), param.numel(),
                                 float(lr), float(beta1), float(beta2), float(eps), int(step),
                                 _lib.stream_handle(param.device))
    _lib.check(rc, "ck_adam_step")
    # written through a raw pointer: bump the version counters so caches keyed
    # on (data_ptr, _version) -- e.g. the layer's coefficient prep -- refresh
    torch.autograd.graph.increment_version(param)
    torch.autograd.graph.increment_version(m)
    torch.autograd.graph.increment_version(v)


def cosine_scale(step_no: int, total_steps: int) -> float:
    """0.5 (1 + cos(pi step / total)) -- network_train's decay (model.py:447-451)."""
    return 0.5 * (1.0 + math.cos(math.pi * step_no / total_steps))


class Adam(torch.optim.Optimizer):
    """torch optimizer front end of ck_adam_step (reference semantics, fp32 state).

    ``step(lr_scale=...)`` multiplies the learning rate for this step only.
    Parameters without a gradient are skipped (their moments stay put), but
    the step counter is shared, as in the reference's AdamState.

    ``capturable=True`` keeps the step counter and the bias corrections on the
    device (ck_adam_begin / ck_adam_step_dev), so a training step captured in
    a CUDA graph advances them on every replay; the learning rate (and
    lr_scale) are then fixed at capture.
    """

    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8, capturable: bool = False):
        if lr < 0.0:
            raise ValueError(f"invalid learning rate: {lr}")
        super().__init__(params, dict(lr=lr, betas=tuple(betas), eps=eps))
        self._step = 0
        self.capturable = capturable
        self._dev_state = {}

    @property
    def step_count(self) -> int:
        return self._step

    def _device_counters(self, group_idx: int, device):
        st = self._dev_state.get((group_idx, device))
        if st is None:
            st = (torch.zeros(1, dtype=torch.int64, device=device), torch.ones(2, dtype=torch.float32, device=device))
            self._dev_state[(group_idx, device)] = st
        return st

    @torch.no_grad()
    def step(self, closure=None, lr_scale: float = 1.0):
        loss = closure() if closure is not None else None
        self._step += 1
        if self.capturable:
            self._step_capturable(lr_scale)
            return loss
        for group in self.param_groups:
            b1, b2 = group["betas"]
            lr = group["lr"] * lr_scale
            for dev, items in self._grouped(group).items():
                self._multi(items, lr, b1, b2, group["eps"], self._step, None, dev)
        return loss

    def _grouped(self, group) -> dict:
        """{device: [(p, g, m, v)]} of the group's parameters with gradients
        (moment buffers created on first use)."""
        out = {}
        for p in group["params"]:
            if p.grad is None:
                continue
            if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
                raise ValueError("Adam: parameters must be contiguous fp32 CUDA tensors")
            st = self.state[p]
            if not st:
                st["m"] = torch.zeros_like(p, memory_format=torch.contiguous_format)
                st["v"] = torch.zeros_like(p, memory_format=torch.contiguous_format)
            g = p.grad if p.grad.is_contiguous() else p.grad.contiguous()
            out.setdefault(p.device, []).append((p, g, st["m"], st["v"]))
        return out

    @staticmethod
    def _multi(items, lr, b1, b2, eps, step, bc, dev) -> None:
        """One ck_adam_step_multi launch for all of a device's tensors."""
        n = len(items)
        arr = lambda k: (ctypes.c_void_p * n)(*[it[k].data_ptr() for it in items])  # noqa: E731
        sizes = (ctypes.c_int64 * n)(*[it[0].numel() for it in items])
        _lib.check(_lib.lib().ck_adam_step_multi(n, arr(0), arr(1), arr(2), arr(3), sizes, float(lr), float(b1),
                                                 float(b2), float(eps), int(step),
                                                 bc.data_ptr() if bc is not None else None,
                                                 _lib.stream_handle(dev)), "ck_adam_step_multi")
        for p, _, m, v in items:
            for t in (p, m, v):
                torch.autograd.graph.increment_version(t)

    def _step_capturable(self, lr_scale: float) -> None:
        lib = _lib.lib()
        for gi, group in enumerate(self.param_groups):
            b1, b2 = group["betas"]
            lr = group["lr"] * lr_scale
            for dev, items in self._grouped(group).items():
                step_t, bc = self._device_counters(gi, dev)
                _lib.check(lib.ck_adam_begin(step_t.data_ptr(), bc.data_ptr(), float(b1), float(b2),
                                             _lib.stream_handle(dev)), "ck_adam_begin")
                self._multi(items, lr, b1, b2, group["eps"], 0, bc, dev)