"""Autograd wrappers of the fused elementwise kernels (libqeft_b200 qeft_rmsnorm_*,
qeft_rope, qeft_silu_mul_*) used by the fine-tuning host model for fp16/bf16
activations. Semantics follow the reference engine (pkg/src/qeft/model.py:249-275
RMS-norm and rotary, 389-391 / 437-438 SwiGLU); the frozen norm gain gets no
gradient (tuning.py: backward_batch(..., param_grads=False))."""

from __future__ import annotations

import torch

from . import _lib
from .layer import _DT

_TDT = {torch.float16: _DT["f16"], torch.bfloat16: _DT["bf16"]}


def supported(x) -> bool:
    return x.is_cuda and x.dtype in _TDT


class _RMSNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gain):
        C = x.shape[-1]
        x2 = x.reshape(-1, C).contiguous()
        y = torch.empty_like(x2)
        rstd = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
        g = gain.float().contiguous()
        _lib.check(_lib.lib().qeft_rmsnorm_fwd(x2.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(),
                                               x2.shape[0], C, _TDT[x.dtype], _lib.stream_ptr()), "rmsnorm_fwd")
        ctx.save_for_backward(x2, g, rstd)
        return y.view(x.shape)

    @staticmethod
    def backward(ctx, dy):
        x2, g, rstd = ctx.saved_tensors
        C = x2.shape[1]
        dy2 = dy.reshape(-1, C).contiguous()
        dx = torch.empty_like(x2)
        _lib.check(_lib.lib().qeft_rmsnorm_bwd(dy2.data_ptr(), x2.data_ptr(), g.data_ptr(), rstd.data_ptr(), None,
                                               dx.data_ptr(), x2.shape[0], C, _TDT[dy2.dtype], _lib.stream_ptr()),
                   "rmsnorm_bwd")
        return dx.view(dy.shape), None


class _ResidualRMSNorm(torch.autograd.Function):
    """(x, rms_norm(x)) for a residual stream x that both continues and feeds a norm: the
    backward is ONE qeft_rmsnorm_bwd with the residual gradient folded in (its dres input),
    instead of the norm's backward plus an autograd add."""

    @staticmethod
    def forward(ctx, x, gain):
        C = x.shape[-1]
        x2 = x.reshape(-1, C).contiguous()
        y = torch.empty_like(x2)
        rstd = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
        g = gain.float().contiguous()
        _lib.check(_lib.lib().qeft_rmsnorm_fwd(x2.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(),
                                               x2.shape[0], C, _TDT[x.dtype], _lib.stream_ptr()), "rmsnorm_fwd")
        ctx.save_for_backward(x2, g, rstd)
        return x.view_as(x), y.view(x.shape)

    @staticmethod
    def backward(ctx, dres, dy):
        x2, g, rstd = ctx.saved_tensors
        C = x2.shape[1]
        if dy is None:
            return dres, None
        dy2 = dy.reshape(-1, C).contiguous()
        dr = dres.reshape(-1, C).contiguous() if dres is not None else None
        if dr is not None and dr.dtype != dy2.dtype:
            dr = dr.to(dy2.dtype)
        dx = torch.empty_like(x2)
        _lib.check(_lib.lib().qeft_rmsnorm_bwd(dy2.data_ptr(), x2.data_ptr(), g.data_ptr(), rstd.data_ptr(),
                                               dr.data_ptr() if dr is not None else None, dx.data_ptr(),
                                               x2.shape[0], C, _TDT[dy2.dtype], _lib.stream_ptr()), "rmsnorm_bwd")
        return dx.view(dy.shape), None


class _Rope(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, cos, sin, T, H, hd):
        xc = x.contiguous()
        y = torch.empty_like(xc)
        rows = xc.numel() // (H * hd)
        _lib.check(_lib.lib().qeft_rope(xc.data_ptr(), y.data_ptr(), cos.data_ptr(), sin.data_ptr(), rows, T, H, hd,
                                        0, _TDT[x.dtype], _lib.stream_ptr()), "rope")
        ctx.save_for_backward(cos, sin)
        ctx.dims = (rows, T, H, hd)
        return y

    @staticmethod
    def backward(ctx, dy):
        cos, sin = ctx.saved_tensors
        rows, T, H, hd = ctx.dims
        dyc = dy.contiguous()
        dx = torch.empty_like(dyc)
        _lib.check(_lib.lib().qeft_rope(dyc.data_ptr(), dx.data_ptr(), cos.data_ptr(), sin.data_ptr(), rows, T, H, hd,
                                        1, _TDT[dy.dtype], _lib.stream_ptr()), "rope_bwd")
        return dx, None, None, None, None, None


class _SiluMul(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, u):
        gc, uc = g.contiguous(), u.contiguous()
        f = torch.empty_like(gc)
        _lib.check(_lib.lib().qeft_silu_mul_fwd(gc.data_ptr(), uc.data_ptr(), f.data_ptr(), gc.numel(),
                                                _TDT[g.dtype], _lib.stream_ptr()), "silu_mul_fwd")
        ctx.save_for_backward(gc, uc)
        return f

    @staticmethod
    def backward(ctx, df):
        gc, uc = ctx.saved_tensors
        dfc = df.contiguous()
        dg, du = torch.empty_like(gc), torch.empty_like(uc)
        _lib.check(_lib.lib().qeft_silu_mul_bwd(dfc.data_ptr(), gc.data_ptr(), uc.data_ptr(), dg.data_ptr(),
                                                du.data_ptr(), gc.numel(), _TDT[gc.dtype], _lib.stream_ptr()),
                   "silu_mul_bwd")
        return dg, du


class _CrossEntropy(torch.autograd.Function):
    """Mean next-token NLL of fp16/bf16 logits (rows, V) in fp32 math, no fp32 copy of the
    logits: qeft_cross_entropy_fwd keeps lse per row; the backward recomputes the softmax."""

    @staticmethod
    def forward(ctx, z, tgt):
        rows, V = z.shape
        zc = z if z.stride(1) == 1 and z.stride(0) % 8 == 0 and z.data_ptr() % 16 == 0 else z.contiguous()
        t = tgt.contiguous().to(torch.int64)
        loss = torch.empty(rows, dtype=torch.float32, device=z.device)
        lse = torch.empty(rows, dtype=torch.float32, device=z.device)
        _lib.check(_lib.lib().qeft_cross_entropy_fwd(zc.data_ptr(), zc.stride(0), rows, V, t.data_ptr(),
                                                     loss.data_ptr(), lse.data_ptr(), _TDT[z.dtype],
                                                     _lib.stream_ptr()), "cross_entropy_fwd")
        ctx.save_for_backward(zc, t, lse)
        return loss.mean()

    @staticmethod
    def backward(ctx, g):
        zc, t, lse = ctx.saved_tensors
        rows, V = zc.shape
        gs = (g.float() / rows).reshape(1).contiguous()
        dz = torch.empty_like(zc)
        _lib.check(_lib.lib().qeft_cross_entropy_bwd(zc.data_ptr(), zc.stride(0), rows, V, t.data_ptr(),
                                                     lse.data_ptr(), gs.data_ptr(), dz.data_ptr(), dz.stride(0),
                                                     _TDT[zc.dtype], _lib.stream_ptr()), "cross_entropy_bwd")
        return dz, None


def cross_entropy(z, tgt):
    """mean_r(logsumexp(z[r]) - z[r, tgt[r]]) for fp16/bf16 CUDA logits (rows, V)."""
    return _CrossEntropy.apply(z, tgt)


def residual_rms_norm(x, gain):
    """(x, rms_norm(x, gain)): use the first output as the continuing residual stream."""
    return _ResidualRMSNorm.apply(x, gain)


def rms_norm(x, gain):
    return _RMSNorm.apply(x, gain)


def rope(x, cos, sin, T, H, hd):
    """x: (B, T, H*hd) token-major; returns the rotated tensor in the same layout."""
    return _Rope.apply(x, cos, sin, T, H, hd)


def silu_mul(g, u):
    return _SiluMul.apply(g, u)


def decode_attention(q, k, v, k_cache, v_cache, cos, sin, pos_dev, H, hd, out=None):
    """Decode step (no autograd): rotary on q/k at *pos_dev, k/v appended to the caches, and the
    query's causal attention over positions 0..pos in one kernel; returns o (B, H*hd)."""
    from .layer import _Workspace
    global _ATTN_WS
    B, T = q.shape[0], k_cache.shape[2]
    o = torch.empty_like(q) if out is None else out
    L = _lib.lib()
    if _ATTN_WS is None:
        _ATTN_WS = _Workspace()  # zero-filled once per (device, stream); the kernel re-arms its counters
    ws = _ATTN_WS.get(int(L.qeft_decode_attention_workspace_bytes(B, H, hd)), q.device)
    _lib.check(L.qeft_decode_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), k_cache.data_ptr(),
                                       v_cache.data_ptr(), cos.data_ptr(), sin.data_ptr(), pos_dev.data_ptr(),
                                       o.data_ptr(), B, H, hd, T, _TDT[q.dtype], ws.data_ptr(), ws.numel(),
                                       _lib.stream_ptr()), "decode_attention")
    return o


_ATTN_WS = None


def rope_kv(q, k, v, q_out, k_cache, v_cache, cos, sin, pos_dev, H, hd):
    """Decode step (no autograd): q_out = rope(q); k_cache/v_cache[:, :, *pos_dev] = rope(k), v.
    q/k/v (B, H*hd); caches (B, H, T, hd); pos_dev a device int64 scalar."""
    B, T = q.shape[0], k_cache.shape[2]
    _lib.check(_lib.lib().qeft_rope_kv(q.data_ptr(), k.data_ptr(), v.data_ptr(), q_out.data_ptr(),
                                       k_cache.data_ptr(), v_cache.data_ptr(), cos.data_ptr(), sin.data_ptr(),
                                       pos_dev.data_ptr(), B, H, hd, T, _TDT[q.dtype], _lib.stream_ptr()),
               "rope_kv")
    return q_out
