"""Torch host of the LLaMA-style decoder whose linears are QEFTLinear layers.

This is the caller of the hot path during fine-tuning: it restates the
reference engine's forward semantics (pkg/src/qeft/model.py:323-407 forward_batch,
RMS-norm 262-266, rotary 249-259, SwiGLU, causal softmax attention, frozen
dense head) in PyTorch, so autograd supplies the backward of the non-linear
parts while every quantized linear runs through libqeft_b200 (QEFTLinear).
Embedding, norm gains and the head are frozen buffers; the only Parameters are
the weak-column fp32 masters, exactly the reference's trainable set
(tuning.py:187-248, backward_batch with param_grads=False).

Layout is token-major (B, T, C) -- the torch orientation; the reference's
(B, C, T) arrays are its transpose. Channel c of a head-split tensor is
h * head_dim + j as in the reference (model.py:372-374).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from . import fused
from .errors import ShapeError
from .qlinear import QEFTLinear, grouped_linear

_GROUPED = __import__("os").environ.get("QEFT_GROUPED", "1") != "0"  # A/B knob
from .qmodel import BLOCK_LINEARS, RMS_EPS, ROPE_BASE, ModelConfig

_TD = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def rope_tables(head_dim: int, n_tokens: int, device):
    """cos/sin (T, head_dim/2) in fp32, from fp64 angles (model.py:249-253)."""
    half = head_dim // 2
    inv_freq = ROPE_BASE ** (-np.arange(half, dtype=np.float64) / half)
    ang = np.outer(np.arange(n_tokens, dtype=np.float64), inv_freq)
    return (torch.from_numpy(np.cos(ang).astype(np.float32)).to(device),
            torch.from_numpy(np.sin(ang).astype(np.float32)).to(device))


def rope_apply(x, cos, sin):
    """x (B, H, T, hd): rotate (first half, second half) pairs (model.py:256-259)."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos.to(x.dtype), sin.to(x.dtype)
    return torch.cat([x1 * c - x2 * s, x1 * s + x2 * c], dim=-1)


def rms_norm(x, gain):
    """gain * x / sqrt(mean(x^2) + eps) over channels (model.py:262-266)."""
    xf = x.float()
    r = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + RMS_EPS)
    return (xf * r * gain.float()).to(x.dtype)


class QEFTBlock(torch.nn.Module):
    def __init__(self, gain1, gain2, layers: dict):
        super().__init__()
        self.register_buffer("gain1", gain1)
        self.register_buffer("gain2", gain2)
        for nm in BLOCK_LINEARS:
            self.add_module(nm, layers[nm])

    def forward(self, x, cos, sin, cfg: ModelConfig):
        if fused.supported(x) and x.shape[-1] % 8 == 0 and cfg.d_ff % 8 == 0:
            return self._forward_fused(x, cos, sin, cfg)
        B, T, _ = x.shape
        H, hd = cfg.n_heads, cfg.head_dim
        a = rms_norm(x, self.gain1)
        q = self.wq(a).to(x.dtype).view(B, T, H, hd).transpose(1, 2)
        k = self.wk(a).to(x.dtype).view(B, T, H, hd).transpose(1, 2)
        v = self.wv(a).to(x.dtype).view(B, T, H, hd).transpose(1, 2)
        q, k = rope_apply(q, cos, sin), rope_apply(k, cos, sin)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True, scale=1.0 / math.sqrt(hd))
        o = o.transpose(1, 2).reshape(B, T, H * hd)
        x1 = x + self.wo(o).to(x.dtype)
        b2 = rms_norm(x1, self.gain2)
        u = self.w_up(b2).to(x.dtype)
        g = self.w_gate(b2).to(x.dtype)
        f = F.silu(g) * u
        return x1 + self.w_down(f).to(x.dtype)

    def _forward_fused(self, x, cos, sin, cfg: ModelConfig):
        """fp16/bf16 activations: RMS-norm, rotary and SwiGLU run as fused libqeft_b200 kernels."""
        B, T, _ = x.shape
        H, hd = cfg.n_heads, cfg.head_dim
        # the residual stream passes through the norm's op, so its gradient joins the norm's
        # backward kernel (no separate add)
        x, a = fused.residual_rms_norm(x, self.gain1)
        # q/k/v (and gate/up) read the same normed input: one grouped op, whose backward sums
        # the three dX in one buffer (GEMM reduce-add epilogue)
        if _GROUPED:
            qp, kp, vp = grouped_linear([self.wq, self.wk, self.wv], a)
        else:
            qp, kp, vp = self.wq(a), self.wk(a), self.wv(a)
        q = fused.rope(qp, cos, sin, T, H, hd).view(B, T, H, hd).transpose(1, 2)
        k = fused.rope(kp, cos, sin, T, H, hd).view(B, T, H, hd).transpose(1, 2)
        v = vp.view(B, T, H, hd).transpose(1, 2)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True, scale=1.0 / math.sqrt(hd))
        x1 = x + self.wo(o.transpose(1, 2).reshape(B, T, H * hd))
        x1, b2 = fused.residual_rms_norm(x1, self.gain2)
        gt, up = grouped_linear([self.w_gate, self.w_up], b2) if _GROUPED else (self.w_gate(b2), self.w_up(b2))
        f = fused.silu_mul(gt, up)
        return x1 + self.w_down(f)


class QEFTDecoder(torch.nn.Module):
    """forward(tokens (B, T) int64) -> logits (B, T, vocab) in the compute dtype."""

    def __init__(self, cfg: ModelConfig, embedding, blocks, final_gain, head, compute_dtype="f32"):
        super().__init__()
        cfg.validate()
        self.cfg = cfg
        self.compute_dtype = _TD[compute_dtype]
        self.register_buffer("embedding", embedding.to(self.compute_dtype))
        self.blocks = torch.nn.ModuleList(blocks)
        self.register_buffer("final_gain", final_gain)
        self.register_buffer("head", head.to(self.compute_dtype))
        self._rope = {}

    # ------------------------------------------------------------------
    @classmethod
    def from_quantized_model(cls, qm, act_dtype="bf16", compute_dtype="f32", device="cuda"):
        """Device model of a QuantizedModel (qmodel.py:47-71 record)."""
        def t(a):
            return torch.as_tensor(np.asarray(a, np.float32)).to(device)
        blocks = []
        for i, b in enumerate(qm.blocks):
            layers = {nm: QEFTLinear.from_quantized(b.layers[nm], dtype=act_dtype, name=f"b{i}.{nm}", device=device)
                      for nm in BLOCK_LINEARS}
            blocks.append(QEFTBlock(t(b.gain1), t(b.gain2), layers))
        return cls(qm.config, t(qm.embedding), blocks, t(qm.final_gain), t(qm.head), compute_dtype)

    @classmethod
    def synthetic(cls, cfg: ModelConfig, *, k=128, bits=4, g=128, act_dtype="bf16",
                  compute_dtype="bf16", seed=0, device="cuda"):
        """Random-init model of the given shape directly in the B200 layout
        (no host quantization): the benchmark model (SURVEY.md 8(d) 7B fine-tune)."""
        from .decode import random_layer
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        d, ff, V = cfg.d_model, cfg.d_ff, cfg.vocab_size
        shapes = {"wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d),
                  "w_up": (ff, d), "w_gate": (ff, d), "w_down": (d, ff)}
        blocks = []
        for i in range(cfg.n_blocks):
            layers = {}
            for j, nm in enumerate(BLOCK_LINEARS):
                oc, ic = shapes[nm]
                dl = random_layer(oc, ic, k, bits, g, act_dtype, seed=seed * 1000003 + i * 7 + j,
                                  device=device)
                layers[nm] = QEFTLinear(dl, name=f"b{i}.{nm}")
            ones = torch.ones(d, device=device)
            blocks.append(QEFTBlock(ones, ones.clone(), layers))
        emb = torch.randn(V, d, device=device, generator=gen) / math.sqrt(d)
        head = torch.randn(V, d, device=device, generator=gen) / math.sqrt(d)
        return cls(cfg, emb, blocks, torch.ones(d, device=device), head, compute_dtype)

    # ------------------------------------------------------------------
    def linears(self):
        for blk in self.blocks:
            for nm in BLOCK_LINEARS:
                yield getattr(blk, nm)

    def rope(self, T, device):
        key = (T, str(device))
        if key not in self._rope:
            self._rope[key] = rope_tables(self.cfg.head_dim, T, device)
        return self._rope[key]

    def forward(self, tokens):
        cfg = self.cfg
        if tokens.dim() != 2:
            raise ShapeError(f"tokens must be (batch, T), got {tuple(tokens.shape)}")
        B, T = tokens.shape
        if T > cfg.max_seq:
            raise ShapeError(f"sequence length {T} exceeds max_seq {cfg.max_seq}")
        cos, sin = self.rope(T, tokens.device)
        x = F.embedding(tokens, self.embedding)
        for blk in self.blocks:
            x = blk(x, cos, sin, cfg)
        z = fused.rms_norm(x, self.final_gain) if fused.supported(x) else rms_norm(x, self.final_gain)
        return z @ self.head.t()

    @torch.no_grad()
    def refresh_weak(self):
        for lin in self.linears():
            lin.refresh()


def cross_entropy_mean(logits, targets):
    """Mean next-token NLL over all positions (model.py:531-547), fp32 softmax. fp16/bf16 CUDA
    logits take the fused kernel (no fp32 copy of the (tokens x vocab) logits)."""
    V = logits.shape[-1]
    if fused.supported(logits) and V % 8 == 0 and V <= 65536:
        return fused.cross_entropy(logits.reshape(-1, V), targets.reshape(-1))
    return F.cross_entropy(logits.float().reshape(-1, V), targets.reshape(-1), reduction="mean")
