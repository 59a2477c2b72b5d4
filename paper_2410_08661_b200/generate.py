"""End-to-end greedy decoding around the GEMV.

The reference's harness `bench_generate` (pkg/src/qeft/kernels.py:197-228) has no KV cache:
each new token recomputes the whole prefix, every linear layer going column by column through
its matvec path. `KVDecoder` is the B200 form of the same greedy loop. Per token and block it runs:
  q/k/v: one qeft_gemv_multi_rmsnorm launch when the three share geometry (the RMS-norm runs
     in its x staging), else RMS-norm + per-layer qeft_gemv
  -> rotary on q/k at the token's position + k/v appended to the cache + attention over
     positions 0..pos, fp32 softmax (one qeft_decode_attention; rope_kv + torch SDPA otherwise)
  -> o (qeft_gemv, irregular / online-reorder layouts gather x in-kernel), the residual add
     fused into its epilogue (QEFT_Y_ACCUMULATE)
  -> gate/up (one launch, RMS-norm in its x staging) -> down over silu(gate)*up (SwiGLU in its
     x staging, qeft_gemv_swiglu), residual fused
The final norm and the frozen dense head follow, then argmax. Semantics follow the reference
engine's forward (model.py:323-407): one decode step at position p equals column p of a full
causal forward. The same greedy token choice (np.argmax: first maximum) is kept.

`capture=True` records one step as a CUDA graph. The position is a device scalar: rotary
rows, the cache write and the attention mask are indexed on device, so one graph serves every
step (attention then spans the preallocated cache, masked past the position).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import decode, fused
from .errors import ShapeError
from .model import QEFTDecoder


def _same_geometry(layers) -> bool:
    """Layers one qeft_gemv_multi launch can serve: same input geometry and column map
    (the C side checks the same fields)."""
    a = layers[0].dl
    return all(d.ic == a.ic and d.k == a.k and d.bits == a.bits and d.g == a.g and d.dtype == a.dtype
               and d.structured_fast == a.structured_fast
               and (a.structured_fast or d.colmap.data_ptr() == a.colmap.data_ptr())
               for d in (l.dl for l in layers[1:]))


class KVDecoder:
    """Incremental decoding of a QEFTDecoder with a preallocated KV cache (batch 1..16)."""

    def __init__(self, model: QEFTDecoder, max_seq: int | None = None, batch: int = 1,
                 capture: bool = False):
        cfg = model.cfg
        self.model, self.cfg = model, cfg
        self.B = batch
        if not 1 <= batch <= 16:
            raise ShapeError("KVDecoder: batch must be 1..16 (decode GEMV columns)")
        self.T = max_seq or cfg.max_seq
        if self.T > cfg.max_seq:
            raise ShapeError(f"max_seq {self.T} exceeds the model's {cfg.max_seq}")
        blk0 = model.blocks[0]
        self.dt = blk0.wq.dl.tdtype
        dev = model.embedding.device
        H, hd = cfg.n_heads, cfg.head_dim
        self.k_cache = [torch.zeros(batch, H, self.T, hd, dtype=self.dt, device=dev) for _ in model.blocks]
        self.v_cache = [torch.zeros_like(c) for c in self.k_cache]
        cos, sin = model.rope(self.T, dev)
        self.cos, self.sin = cos.contiguous(), sin.contiguous()
        self.qkv_fused = [_same_geometry([b.wq, b.wk, b.wv]) for b in model.blocks]
        self.gu_fused = [_same_geometry([b.w_gate, b.w_up]) for b in model.blocks]
        self.emb = model.embedding.to(self.dt)
        self.head = model.head.to(self.dt)
        self.pos_dev = torch.zeros((), dtype=torch.int64, device=dev)
        self.tok_dev = torch.zeros(batch, dtype=torch.int64, device=dev)
        self.graph = None
        self.capture = capture

    # ------------------------------------------------------------------ one step
    def _step(self, tok, pos):
        """tok (B,) int64 on device; pos: python int, or the device scalar under capture."""
        cfg, B = self.cfg, self.B
        H, hd = cfg.n_heads, cfg.head_dim
        dyn = isinstance(pos, torch.Tensor)
        x = F.embedding(tok, self.emb).contiguous()  # (B, d) residual stream, updated in place
        if dyn and hd != 128:
            # additive mask (0 / -inf) built once per step: a boolean mask would be converted
            # (fill + masked_fill) inside every block's attention call
            keep = torch.zeros(1, 1, 1, self.T, dtype=self.dt, device=tok.device).masked_fill_(
                (torch.arange(self.T, device=tok.device) > pos).view(1, 1, 1, self.T), float("-inf"))
        for i, blk in enumerate(self.model.blocks):
            if self.qkv_fused[i]:
                # the RMS-norm runs inside the q/k/v launch's x staging
                q = torch.empty(B, blk.wq.oc, dtype=self.dt, device=x.device)
                k, v = torch.empty_like(q), torch.empty(B, blk.wv.oc, dtype=self.dt, device=x.device)
                decode.gemv_multi([blk.wq.dl, blk.wk.dl, blk.wv.dl], x, [q, k, v], norm_gain=blk.gain1)
            else:
                a = fused.rms_norm(x, blk.gain1)
                q, k, v = blk.wq.dl.gemv(a), blk.wk.dl.gemv(a), blk.wv.dl.gemv(a)
            kc, vc = self.k_cache[i], self.v_cache[i]
            if dyn and hd == 128:
                # rotary + cache append + attention over positions 0..pos, one kernel
                o2 = fused.decode_attention(q, k, v, kc, vc, self.cos, self.sin, self.pos_dev, H, hd)
            else:
                # rotary on q and k + the cache append at the device position, one kernel
                qr = fused.rope_kv(q, k, v, torch.empty_like(q), kc, vc, self.cos, self.sin, self.pos_dev, H, hd)
                qh = qr.view(B, H, 1, hd)
                if dyn:
                    o = F.scaled_dot_product_attention(qh, kc, vc, attn_mask=keep, scale=1.0 / math.sqrt(hd))
                else:
                    o = F.scaled_dot_product_attention(qh, kc[:, :, :pos + 1], vc[:, :, :pos + 1],
                                                       scale=1.0 / math.sqrt(hd))
                o2 = o.transpose(1, 2).reshape(B, H * hd)
            x = x.contiguous()
            blk.wo.dl.gemv(o2, out=x, accumulate=True)  # x += Wo o
            if self.gu_fused[i]:
                gt = torch.empty(B, blk.w_gate.oc, dtype=self.dt, device=x.device)
                up = torch.empty_like(gt)
                decode.gemv_multi([blk.w_gate.dl, blk.w_up.dl], x, [gt, up], norm_gain=blk.gain2)
            else:
                b2 = fused.rms_norm(x, blk.gain2)
                gt, up = blk.w_gate.dl.gemv(b2), blk.w_up.dl.gemv(b2)
            blk.w_down.dl.gemv_swiglu(gt, up, out=x, accumulate=True)  # x += Wdown (silu(gt) * up)
        z = fused.rms_norm(x, self.model.final_gain)
        return (z @ self.head.t()).float()  # (B, V) fp32 logits

    @torch.no_grad()
    def step(self, tok, pos: int):
        """Logits (B, V) for tokens `tok` (B,) at position `pos` (appends to the cache)."""
        if not 0 <= pos < self.T:
            raise ShapeError(f"position {pos} outside the cache (max_seq {self.T})")
        tok = torch.as_tensor(tok, dtype=torch.int64).view(self.B)
        self.pos_dev.fill_(pos)  # read on device by the rotary + cache-append kernel
        if not self.capture:
            return self._step(tok.to(self.tok_dev.device), pos)
        self.tok_dev.copy_(tok, non_blocking=True)
        if self.graph is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._step(self.tok_dev, self.pos_dev)  # warm-up: workspaces, cuDNN plans
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.out = self._step(self.tok_dev, self.pos_dev)
            # the capture itself did not run the step: replay it
        self.graph.replay()
        return self.out

    def reset(self):
        for c in self.k_cache + self.v_cache:
            c.zero_()


@dataclass
class GenerationResult:
    """kernels.py:189-194."""
    tokens: np.ndarray
    stats: dict = field(default_factory=dict)
    tokens_per_s: float = 0.0
    elapsed_ns: int = 0


def generate(dec: KVDecoder, prompt, n_tokens: int) -> GenerationResult:
    """Greedy batch-1 generation: prompt tokens fill the cache step by step, then n_tokens are
    chosen by argmax (first maximum, as np.argmax). Timing covers the generated tokens."""
    prompt = np.asarray(prompt, dtype=np.int64)
    if prompt.ndim != 1 or prompt.size == 0:
        raise ShapeError("prompt must be a nonempty 1-D token sequence")
    if prompt.size + n_tokens > dec.T:
        raise ShapeError(f"prompt ({prompt.size}) + n_tokens ({n_tokens}) exceeds max_seq {dec.T}")
    if dec.B != 1:
        raise ShapeError("generate() is batch 1 (bench_generate semantics)")
    dec.reset()
    logits = None
    for p, t in enumerate(prompt):
        logits = dec.step(torch.tensor([int(t)]), p)
    out = []
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    pos = prompt.size
    for _ in range(n_tokens):
        nxt = int(torch.argmax(logits[0]))
        out.append(nxt)
        if len(out) == n_tokens:
            break
        logits = dec.step(torch.tensor([nxt]), pos)
        pos += 1
    torch.cuda.synchronize()
    el = time.perf_counter_ns() - t0
    return GenerationResult(tokens=np.array(out, np.int64), tokens_per_s=n_tokens / (el / 1e9) if el else 0.0,
                            elapsed_ns=el)


def bench_generate(model, prompt, n_tokens: int, reference: bool = False, repeats: int = 1,
                   act_dtype: str = "f16", capture: bool = True) -> GenerationResult:
    """kernels.py:197-228 on the B200 path: greedy batch-1 generation, median-throughput run.
    `model` is a QuantizedModel (repacked to the device once) or a QEFTDecoder."""
    if reference:
        raise ShapeError("reference=True is the reference's own CPU path; use the reference package")
    if not isinstance(model, QEFTDecoder):
        model = QEFTDecoder.from_quantized_model(model, act_dtype=act_dtype, compute_dtype=act_dtype)
    dec = KVDecoder(model, capture=capture)
    runs = sorted((generate(dec, prompt, n_tokens) for _ in range(max(1, repeats))),
                  key=lambda r: r.tokens_per_s)
    return runs[len(runs) // 2]
