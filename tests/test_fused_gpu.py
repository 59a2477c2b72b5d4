"""Fused elementwise kernels of the fine-tuning host model vs fp32 torch restatements of the
reference engine (pkg/src/qeft/model.py:249-275 RMS-norm / rotary, 389-391 and 437-438 SwiGLU),
forward and backward. Tolerance: bf16 storage, max|d| / max(1, max|ref|) <= 1e-2."""

import math

import numpy as np
import pytest

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _np(t):
    return t.detach().float().cpu().numpy()


@pytest.mark.parametrize("dt", ["bf16", "f16"])
def test_rmsnorm_fwd_bwd(torch_, dt):
    torch = torch_
    from paper_2410_08661_b200 import fused
    td = {"bf16": torch.bfloat16, "f16": torch.float16}[dt]
    x = torch.randn(3, 37, 4096, device="cuda").to(td).requires_grad_(True)
    gain = 1.0 + 0.1 * torch.randn(4096, device="cuda")
    y = fused.rms_norm(x, gain)
    xr = x.detach().float().requires_grad_(True)
    yr = gain * xr / torch.sqrt((xr * xr).mean(-1, keepdim=True) + 1e-5)
    assert rel_err(_np(y), _np(yr)) <= 1e-2
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy.float())
    assert rel_err(_np(x.grad), _np(xr.grad)) <= 1e-2


@pytest.mark.parametrize("hd", [128, 8, 6])  # 16-byte vector path, then the per-pair path
def test_rope_fwd_bwd(torch_, hd):
    torch = torch_
    from paper_2410_08661_b200 import fused
    from paper_2410_08661_b200.model import rope_tables
    B, T, H = 2, 65, 4
    cos, sin = rope_tables(hd, T, "cuda")
    x = torch.randn(B, T, H * hd, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = fused.rope(x, cos, sin, T, H, hd)
    xr = x.detach().float().view(B, T, H, hd).requires_grad_(True)
    half = hd // 2
    c, s = cos[None, :, None, :], sin[None, :, None, :]
    x1, x2 = xr[..., :half], xr[..., half:]
    yr = torch.cat([x1 * c - x2 * s, x1 * s + x2 * c], -1)
    assert rel_err(_np(y), _np(yr.reshape(B, T, H * hd))) <= 1e-2
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy.float().view(B, T, H, hd))
    assert rel_err(_np(x.grad), _np(xr.grad.reshape(B, T, H * hd))) <= 1e-2


def test_silu_mul_fwd_bwd(torch_):
    torch = torch_
    from paper_2410_08661_b200 import fused
    g = (2 * torch.randn(77, 11008, device="cuda")).to(torch.bfloat16).requires_grad_(True)
    u = torch.randn(77, 11008, device="cuda").to(torch.bfloat16).requires_grad_(True)
    f = fused.silu_mul(g, u)
    gr = g.detach().float().requires_grad_(True)
    ur = u.detach().float().requires_grad_(True)
    fr = gr * torch.sigmoid(gr) * ur
    assert rel_err(_np(f), _np(fr)) <= 1e-2
    df = torch.randn_like(f)
    f.backward(df)
    fr.backward(df.float())
    assert rel_err(_np(g.grad), _np(gr.grad)) <= 1e-2
    assert rel_err(_np(u.grad), _np(ur.grad)) <= 1e-2


def test_block_fused_matches_torch_path(torch_):
    """One decoder block on the fused path vs the same block through the plain torch
    ops (fp32 non-linear math), bf16 QEFT linears in both."""
    torch = torch_
    from paper_2410_08661_b200 import fused
    from paper_2410_08661_b200.model import QEFTDecoder
    from paper_2410_08661_b200.qmodel import ModelConfig
    cfg = ModelConfig(d_model=512, n_heads=4, head_dim=128, d_ff=1024, n_blocks=1, vocab_size=300, max_seq=256)
    m = QEFTDecoder.synthetic(cfg, k=128, bits=4, g=128, act_dtype="bf16", compute_dtype="bf16", seed=3)
    tok = torch.randint(0, 300, (2, 96), device="cuda")
    blk = m.blocks[0]
    x = torch.randn(2, 96, 512, device="cuda").to(torch.bfloat16)
    cos, sin = m.rope(96, x.device)
    y_f = blk._forward_fused(x, cos, sin, cfg)
    orig = fused.supported
    fused.supported = lambda t: False
    try:
        y_t = blk(x.float(), cos, sin, cfg)
    finally:
        fused.supported = orig
    assert rel_err(_np(y_f), _np(y_t)) <= 2e-2


@pytest.mark.parametrize("dt,rows,V", [("f16", 64, 32000), ("bf16", 33, 1000), ("f16", 5, 8)])
def test_cross_entropy_matches_fp32_torch(dt, rows, V):
    """Fused CE (qeft_cross_entropy_fwd/bwd) against F.cross_entropy on the fp32 image of the
    same logits (the reference's fp32 log-softmax NLL, model.py:531-547): loss to 1e-5
    relative, gradient to one output rounding of the logits' dtype."""
    import torch
    import torch.nn.functional as F
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import fused
    td = torch.float16 if dt == "f16" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(rows + V)
    z = (torch.randn(rows, V, device="cuda", generator=g) * 3).to(td).requires_grad_(True)
    t = torch.randint(0, V, (rows,), device="cuda", generator=g)
    loss = fused.cross_entropy(z, t)
    loss.backward(torch.tensor(1.7, device="cuda"))
    zr = z.detach().float().requires_grad_(True)
    ref = F.cross_entropy(zr, t, reduction="mean")
    (ref * 1.7).backward()
    assert abs(float(loss) - float(ref)) <= 1e-5 * abs(float(ref))
    ulp = 2.0 ** -10 if dt == "f16" else 2.0 ** -7
    err = (z.grad.float() - zr.grad.to(td).float()).abs().max()
    assert float(err) <= ulp * float(zr.grad.abs().max()) + 1e-7


@pytest.mark.parametrize("dt,B,pos", [("f16", 1, 0), ("f16", 1, 600), ("bf16", 2, 77)])
def test_decode_attention_matches_rope_kv_sdpa(dt, B, pos):
    """qeft_decode_attention (rotary + cache append + causal attention over 0..pos, one kernel)
    against qeft_rope_kv + torch SDPA on a copy of the same caches: identical cache rows, and
    the output within one fp16/bf16 rounding of the fp32 softmax attention."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import fused
    from paper_2410_08661_b200.model import rope_tables
    td = torch.float16 if dt == "f16" else torch.bfloat16
    H, hd, T = 32, 128, 641
    g = torch.Generator(device="cuda").manual_seed(pos + B)
    q, k, v = [(torch.randn(B, H * hd, device="cuda", generator=g)).to(td) for _ in range(3)]
    kc = (torch.randn(B, H, T, hd, device="cuda", generator=g)).to(td)
    vc = (torch.randn(B, H, T, hd, device="cuda", generator=g)).to(td)
    kc2, vc2 = kc.clone(), vc.clone()
    cos, sin = rope_tables(hd, T, "cuda")
    p = torch.tensor(pos, dtype=torch.int64, device="cuda")
    o = fused.decode_attention(q, k, v, kc, vc, cos, sin, p, H, hd)
    qr = fused.rope_kv(q, k, v, torch.empty_like(q), kc2, vc2, cos, sin, p, H, hd)
    ref = torch.nn.functional.scaled_dot_product_attention(
        qr.view(B, H, 1, hd).float(), kc2[:, :, :pos + 1].float(), vc2[:, :, :pos + 1].float(),
        scale=1.0 / math.sqrt(hd)).transpose(1, 2).reshape(B, H * hd)
    torch.cuda.synchronize()
    assert torch.equal(kc, kc2) and torch.equal(vc, vc2)
    ulp = 2.0 ** -10 if dt == "f16" else 2.0 ** -7
    err = (o.float() - ref).abs().max()
    assert float(err) <= 2 * ulp * float(ref.abs().max()) + 1e-3, float(err)


def test_residual_rms_norm_folds_the_residual_gradient(torch_):
    """fused.residual_rms_norm: (x, norm(x)) whose backward is one rmsnorm_bwd with the
    residual-path gradient folded in -- equal to rms_norm + an explicit residual add (fp32 sum
    of the two fp16 terms rounded once vs twice: within one fp16 rounding)."""
    torch = torch_
    from paper_2410_08661_b200 import fused
    x = torch.randn(2, 33, 4096, device="cuda").half().requires_grad_(True)
    gain = 1.0 + 0.1 * torch.randn(4096, device="cuda")
    d_res = torch.randn_like(x)
    d_norm = torch.randn_like(x)
    xp, y = fused.residual_rms_norm(x, gain)
    assert xp.data_ptr() == x.data_ptr() and torch.equal(y, fused.rms_norm(x.detach(), gain))
    torch.autograd.backward([xp, y], [d_res, d_norm])
    x2 = x.detach().clone().requires_grad_(True)
    torch.autograd.backward([x2, fused.rms_norm(x2, gain)], [d_res, d_norm])
    scale = float(x2.grad.float().abs().max())
    assert float((x.grad.float() - x2.grad.float()).abs().max()) <= 2 * 2.0 ** -10 * scale


def test_grouped_linear_matches_separate_layers(torch_):
    """qlinear.grouped_linear (q/k/v-style: one op, dX summed by the GEMM's reduce-add epilogue,
    one dW launch) against the three QEFTLinear layers applied separately: same outputs, dX within
    fp16 rounding of the summation order, dW_weak to fp32 summation order."""
    torch = torch_
    from paper_2410_08661_b200.decode import random_layer
    from paper_2410_08661_b200.qlinear import QEFTLinear, grouped_linear
    mods = [QEFTLinear(random_layer(oc, 1024, 128, 4, 128, "f16", seed=s), name=f"l{s}")
            for s, oc in enumerate((512, 512, 256))]
    x = torch.randn(300, 1024, device="cuda").half().requires_grad_(True)
    dys = [torch.randn(300, m.oc, device="cuda").half() for m in mods]
    ys = grouped_linear(mods, x)
    torch.autograd.backward(ys, dys)
    dx_g = x.grad.clone()
    dw_g = [m.weak32.grad.clone() for m in mods]
    for m in mods:
        m.weak32.grad = None
    x.grad = None
    ys2 = [m(x) for m in mods]
    for a_, b_ in zip(ys, ys2):
        assert torch.equal(a_, b_)
    torch.autograd.backward(ys2, dys)
    scale = float(x.grad.float().abs().max())
    assert float((dx_g.float() - x.grad.float()).abs().max()) <= 4 * 2.0 ** -10 * scale
    for a_, m in zip(dw_g, mods):
        assert rel_err(_np(a_), _np(m.weak32.grad)) <= 1e-5
