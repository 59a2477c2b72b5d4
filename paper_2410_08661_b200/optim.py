"""Weak-column optimizer on the GPU (reference API: AdamState, adam_step, and the
global-norm clip of the fine-tune loop, pkg/src/qeft/tuning.py:137-160, 226-236).

`FlatAdam` owns one flat fp32 master / grad / m / v bucket covering every
layer's weak block, so clip + Adam is two fused launches per step regardless
of layer count, and the DP all-reduce is one NCCL call over `grad`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DivergenceError


def _f32(v: float) -> float:
    return float(np.float32(v))


def adam_constants(step: int, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """fp32 images of the reference's Python scalars (tuning.py:154-159)."""
    return dict(lr=_f32(lr), c_b1=_f32(beta1), c_1mb1=_f32(1.0 - beta1), c_b2=_f32(beta2),
                c_1mb2=_f32(1.0 - beta2), bc1=_f32(1.0 - beta1 ** step),
                bc2=_f32(1.0 - beta2 ** step), eps=_f32(eps))


@dataclass
class AdamState:
    """Moments for one weak block (CUDA fp32 tensors) + step counter."""
    m: object
    v: object
    step: int = 0

    @classmethod
    def like(cls, w):
        import torch
        return cls(m=torch.zeros_like(w, dtype=torch.float32), v=torch.zeros_like(w, dtype=torch.float32))


class _Scratch:
    def __init__(self):
        self.t = {}

    def get(self, device):
        import torch
        k = str(device)
        if k not in self.t:
            self.t[k] = (torch.zeros(4096, dtype=torch.float64, device=device),
                         torch.zeros(1, dtype=torch.float64, device=device),
                         torch.zeros(1, dtype=torch.int32, device=device))
        return self.t[k]


_SCRATCH = _Scratch()


def grad_sqnorm(g, out=None):
    """sum(g^2) in fp64 on device (deterministic)."""
    scratch, sq, _ = _SCRATCH.get(g.device)
    out = sq if out is None else out
    _lib.check(_lib.lib().qeft_grad_sqnorm(_lib.ptr(g), g.numel(), _lib.ptr(scratch), _lib.ptr(out),
                                           _lib.stream_ptr()), "grad_sqnorm")
    return out


def div_(g, divisor: float):
    _lib.check(_lib.lib().qeft_div_scalar(_lib.ptr(g), g.numel(), _f32(divisor), _lib.stream_ptr()),
               "div_scalar")
    return g


def adam_clip_(w, m, v, g, step: int, lr, *, max_norm=0.0, beta1=0.9, beta2=0.999, eps=1e-8,
               sqnorm=None, flag=None):
    """In-place clip (by the global norm in `sqnorm`) + Adam on flat fp32 tensors."""
    _, sq, fl = _SCRATCH.get(g.device)
    if sqnorm is None:
        sqnorm = grad_sqnorm(g)
    flag = fl if flag is None else flag
    c = adam_constants(step, lr, beta1, beta2, eps)
    _lib.check(_lib.lib().qeft_adam_clip(
        _lib.ptr(w), _lib.ptr(m), _lib.ptr(v), _lib.ptr(g), g.numel(), _lib.ptr(sqnorm),
        float(max_norm or 0.0), c["lr"], c["c_b1"], c["c_1mb1"], c["c_b2"], c["c_1mb2"], c["bc1"],
        c["bc2"], c["eps"], _lib.ptr(flag), _lib.stream_ptr()), "adam_clip")
    return flag


def adam_step(state: AdamState, w, grad, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Reference signature (tuning.py:148-160): bias-corrected Adam in place on w.
    Raises DivergenceError on a non-finite gradient (nothing is updated)."""
    import torch
    _lib.require_cuda(w, "w")
    _, _, fl = _SCRATCH.get(w.device)
    fl.zero_()
    state.step += 1
    g = grad.contiguous().float()
    adam_clip_(w, state.m, state.v, g, state.step, lr, beta1=beta1, beta2=beta2, eps=eps, flag=fl)
    if int(fl.item()):
        state.step -= 1
        raise DivergenceError("non-finite gradient in adam_step")
    return w


def grad_sqnorm_div(g, divisor: float, out):
    """out = sum((g / divisor)^2), fp64, g / divisor rounded to fp32 first (tuning.py:228-230)."""
    scratch, _, _ = _SCRATCH.get(g.device)
    _lib.check(_lib.lib().qeft_grad_sqnorm_div(_lib.ptr(g), g.numel(), _f32(divisor), _lib.ptr(scratch),
                                               _lib.ptr(out), _lib.stream_ptr()), "grad_sqnorm_div")
    return out


def adam_step_flat(w, m, v, g, descs, n_layers, max_rows, divisor, step, lr, *, max_norm, sqnorm, flag,
                   beta1=0.9, beta2=0.999, eps=1e-8):
    """One fused pass: g / divisor -> global clip -> fp32 Adam -> weak16 shadows."""
    c = adam_constants(step, lr, beta1, beta2, eps)
    _lib.check(_lib.lib().qeft_adam_step_flat(
        _lib.ptr(w), _lib.ptr(m), _lib.ptr(v), _lib.ptr(g), _lib.ptr(descs), n_layers, max_rows, _f32(divisor),
        _lib.ptr(sqnorm), float(max_norm or 0.0), c["lr"], c["c_b1"], c["c_1mb1"], c["c_b2"], c["c_1mb2"],
        c["bc1"], c["bc2"], c["eps"], _lib.ptr(flag), _lib.stream_ptr()), "adam_step_flat")
    return flag


def shadow_descs(layers, offsets):
    """Device array of qeft_shadow_desc_t for FlatAdam.refresh."""
    import torch
    arr = (_lib.ShadowDescT * len(layers))()
    mx = 0
    for i, (dl, off) in enumerate(zip(layers, offsets)):
        arr[i].offset, arr[i].oc, arr[i].k, arr[i].k_pad = off, dl.oc, dl.k, dl.k_pad
        arr[i].act_dtype = 0 if dl.dtype == "f16" else 1
        arr[i].weak16 = dl.weak16.data_ptr()
        mx = max(mx, dl.oc * dl.k)
    raw = torch.frombuffer(bytearray(ctypes.string_at(arr, ctypes.sizeof(arr))), dtype=torch.uint8)
    return raw.cuda(), mx


def refresh_shadows(w32_flat, desc_dev, n_layers, max_elems):
    _lib.check(_lib.lib().qeft_weak_shadow(_lib.ptr(w32_flat), _lib.ptr(desc_dev), n_layers,
                                           max_elems, _lib.stream_ptr()), "weak_shadow")
