"""QEFTLinear: the structured mixed-precision linear layer as a torch module.

Forward is y = x W_hat^T with W_hat = [dequant(codes) | W_weak] in the layer's
own column order (quantizer.py:95-100); backward gives dX through the full
W_hat and dW only for the weak block, computed from the saved weak slice of
the input (the reference's qlinear_forward_train / qlinear_backward,
pkg/src/qeft/tuning.py:52-103). Every product runs in libqeft_b200:
  inference, T <= 16 tokens -> decode GEMV (qeft_gemv)
  otherwise                 -> tcgen05 GEMM (qeft_gemm_fwd); training always takes the GEMM,
                               whose dequantized weights are exactly the dX GEMM's
  backward        -> qeft_gemm_dgrad + qeft_gemm_wgrad_weak
The fp32 master of the weak block is the module's only Parameter; its .grad is
a view into the owner's flat gradient bucket when one is attached (the DP step
all-reduces that bucket in one call), and the fp16/bf16 kernel copy (weak16)
is refreshed from the master after each optimizer step.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .errors import ShapeError
from .layer import DeviceLayer, _DT


class _QEFTLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2, weak32, mod, use_gemv):
        dl: DeviceLayer = mod.dl
        y = dl.gemv(x2) if use_gemv else dl.gemm_fwd(x2)
        ctx.mod = mod
        if weak32.requires_grad and dl.k:
            ctx.save_for_backward(_weak_slice(dl, x2))
        else:
            ctx.save_for_backward(None)
        return y

    @staticmethod
    def backward(ctx, dy):
        mod = ctx.mod
        dl: DeviceLayer = mod.dl
        (xw,) = ctx.saved_tensors
        dy = dy.contiguous()
        if dy.dtype != dl.tdtype:
            dy = dy.to(dl.tdtype)
        dx = dl.gemm_dgrad(dy) if ctx.needs_input_grad[0] else None
        if xw is not None:
            w = mod.weak32
            if w.grad is None:
                w.grad = torch.zeros_like(w)
            # accumulate straight into the (bucket-backed) .grad: micro-batches add up
            # exactly like the reference's acc[name] += grads[name] (tuning.py:219-224)
            dl.gemm_wgrad_weak(dy, xw, out=w.grad, accumulate=True)
            if mod.grad_ready_hook is not None:  # e.g. launch this layer group's DP all-reduce
                mod.grad_ready_hook(mod)
        return dx, None, None, None


class _QEFTGroupFn(torch.autograd.Function):
    """Several QEFT layers over the same input (a block's q/k/v, or gate/up): one forward GEMM
    per layer; the backward sums their dX in place (qeft_gemm_dgrad accumulate, a TMA
    reduce-add in the epilogue) instead of one autograd add per extra consumer of x."""

    @staticmethod
    def forward(ctx, x2, mods, *weaks):
        ys, saved, idx = [], [], []
        for i, (mod, w) in enumerate(zip(mods, weaks)):
            dl: DeviceLayer = mod.dl
            ys.append(dl.gemm_fwd(x2))
            if w.requires_grad and dl.k:
                saved.append(_weak_slice(dl, x2))
                idx.append(i)
        ctx.mods, ctx.widx = mods, idx
        ctx.save_for_backward(*saved)
        return tuple(ys)

    @staticmethod
    def backward(ctx, *dys):
        xws = dict(zip(ctx.widx, ctx.saved_tensors))
        dx = None
        wg = []  # (mod, dy, x_weak) of the layers with a trainable weak block
        for i, (mod, dy) in enumerate(zip(ctx.mods, dys)):
            if dy is None:
                continue
            dl: DeviceLayer = mod.dl
            dy = dy.contiguous()
            if dy.dtype != dl.tdtype:
                dy = dy.to(dl.tdtype)
            if ctx.needs_input_grad[0]:
                dx = dl.gemm_dgrad(dy) if dx is None else dl.gemm_dgrad(dy, out=dx, accumulate=True)
            if i in xws:
                wg.append((mod, dy, xws[i]))
        if wg:
            for mod, _, _ in wg:
                if mod.weak32.grad is None:
                    mod.weak32.grad = torch.zeros_like(mod.weak32)
            xw = wg[0][2]
            same = all(w[2].data_ptr() == xw.data_ptr() and w[0].dl.k == wg[0][0].dl.k for w in wg)
            if len(wg) > 1 and same and all(w[1].stride(0) % 8 == 0 for w in wg) and xw.stride(0) % 8 == 0:
                # every dW_weak of the group in one launch (they share the weak input columns)
                L = _lib.lib()
                n = len(wg)
                arr = (ctypes.POINTER(_lib.QeftLinearT) * n)(*[w[0].dl.cptr for w in wg])
                dyp = (ctypes.c_void_p * n)(*[w[1].data_ptr() for w in wg])
                ldd = (ctypes.c_int64 * n)(*[w[1].stride(0) for w in wg])
                dwp = (ctypes.c_void_p * n)(*[w[0].weak32.grad.data_ptr() for w in wg])
                _lib.check(L.qeft_gemm_wgrad_weak_multi(ctypes.cast(arr, ctypes.c_void_p), n, ctypes.cast(dyp, ctypes.c_void_p),
                                                        ctypes.cast(ldd, ctypes.c_void_p), xw.data_ptr(), xw.stride(0),
                                                        ctypes.cast(dwp, ctypes.c_void_p), wg[0][1].shape[0], 1,
                                                        _lib.stream_ptr()), "gemm_wgrad_weak_multi")
            else:
                for mod, dy, x_w in wg:
                    mod.dl.gemm_wgrad_weak(dy, x_w, out=mod.weak32.grad, accumulate=True)
            for mod, _, _ in wg:
                if mod.grad_ready_hook is not None:
                    mod.grad_ready_hook(mod)
        return (dx, None) + (None,) * len(ctx.mods)


def grouped_linear(mods, x):
    """(mod(x) for mod in mods) for QEFTLinear layers sharing the input x (..., ic); the
    training path takes _QEFTGroupFn (summed dX in one buffer), inference on <= 16 tokens each
    layer's decode GEMV."""
    ic = mods[0].ic
    if any(m.ic != ic or m.dl.tdtype != mods[0].dl.tdtype for m in mods) or x.shape[-1] != ic:
        raise ShapeError("grouped_linear: layers must share the input width and dtype")
    lead = x.shape[:-1]
    x2 = x.reshape(-1, ic)
    if x2.dtype != mods[0].dl.tdtype:
        x2 = x2.to(mods[0].dl.tdtype)
    grad = torch.is_grad_enabled() and (x2.requires_grad or any(m.weak32.requires_grad for m in mods))
    if not grad and x2.shape[0] <= 16:
        return [m(x) for m in mods]
    ys = _QEFTGroupFn.apply(x2, tuple(mods), *[m.weak32 for m in mods])
    return [y.reshape(*lead, m.oc) for y, m in zip(ys, mods)]


_WEAK_VIEW = os.environ.get("QEFT_WEAK_VIEW", "1") != "0"  # A/B knob: 0 = always gather


def _weak_slice(dl: DeviceLayer, x2):
    """x_weak for the backward (TrainableLayerState.x_weak, tuning.py:30-34, 70-71). Structured
    layers hold their weak block in the trailing input columns [m, ic): the wgrad GEMM reads
    that strided view of x in place by TMA (row pitch ic), so no copy is made and no kernel
    launched -- the role the GEMM epilogue would otherwise play. Other layouts gather the k
    weak columns (one small launch)."""
    if (_WEAK_VIEW and dl.structured_fast and x2.stride(1) == 1 and x2.stride(0) % 8 == 0 and dl.m % 8 == 0
            and x2.data_ptr() % 16 == 0 and x2.shape[0] > 1):
        return x2[:, dl.m:dl.m + dl.k]
    return dl.gather_weak(x2)


class QEFTLinear(torch.nn.Module):
    """A QuantizedLinear (or synthetic B200-layout layer) as an nn.Module."""

    def __init__(self, dl: DeviceLayer, name: str = "", trainable: bool = True):
        super().__init__()
        self.dl = dl
        self.name = name
        self.oc, self.ic, self.k = dl.oc, dl.ic, dl.k
        w = dl.weak32
        if w is None:
            # synthetic layers carry only the kernel copy: untile weak16 ([oc_pad/16][k_pad/64]
            # tiles of 16 x 64, csrc/qeft_common.cuh weak_off) into the fp32 master
            kp = dl.k_pad
            w = (dl.weak16.reshape(dl.oc_pad // 16, kp // 64, 16, 64).permute(0, 2, 1, 3)
                 .reshape(dl.oc_pad, kp)[:dl.oc, :dl.k].float().contiguous())
        self.weak32 = torch.nn.Parameter(w.reshape(dl.oc, dl.k).float(), requires_grad=trainable)
        self.grad_ready_hook = None  # called after this layer's dW_weak lands in .grad

    @classmethod
    def from_quantized(cls, q, dtype="bf16", name="", trainable=True, device="cuda"):
        return cls(DeviceLayer.from_quantized(q, dtype=dtype, device=device), name=name, trainable=trainable)

    def forward(self, x):
        if x.shape[-1] != self.ic:
            raise ShapeError(f"{self.name}: input width {x.shape[-1]} != IC {self.ic}")
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.ic)
        if x2.dtype != self.dl.tdtype:
            x2 = x2.to(self.dl.tdtype)
        # inference on <= 16 tokens: the decode GEMV; training: the GEMM (the dX GEMM's weights)
        use_gemv = x2.shape[0] <= 16 and not (torch.is_grad_enabled() and
                                              (self.weak32.requires_grad or x2.requires_grad))
        y = _QEFTLinearFn.apply(x2, self.weak32, self, use_gemv)
        return y.reshape(*lead, self.oc)

    @torch.no_grad()
    def refresh(self):
        """Re-pack the kernel's weak16 from the fp32 master (after an update)."""
        if self.k:
            _lib.check(_lib.lib().qeft_pack_weak(self.weak32.data_ptr(), self.oc, self.k,
                                                 _DT[self.dl.dtype], self.dl.weak16.data_ptr(),
                                                 _lib.stream_ptr()), "pack_weak")

    def extra_repr(self):
        return (f"oc={self.oc}, ic={self.ic}, k={self.k}, bits={self.dl.bits}, g={self.dl.g}, "
                f"dtype={self.dl.dtype}")


def _weak_columns(dl: DeviceLayer):
    """Input columns of the weak block, from the colmap (B200 K order -> column)."""
    cm = dl.colmap[dl.m_pad:dl.m_pad + dl.k].long()
    return cm
