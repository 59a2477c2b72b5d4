"""QEFTLinear (torch autograd over the libqeft_b200 kernels) against an fp64
product with the device-dequantized weights: forward (GEMV for T <= 16, GEMM
above), dX, and dW of the weak block only (tuning.py:52-103).
Tolerance: max|d| / max(1, max|ref|) <= 1e-2 (north_star)."""

import numpy as np
import pytest

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import quantizer
    return quantizer


CASES = [
    # oc, ic, k, bits, g, dtype, T, layout, perm
    (256, 512, 128, 4, 128, "bf16", 1, "structured", False),
    (256, 512, 128, 4, 128, "bf16", 300, "structured", False),
    (300, 768, 64, 3, 64, "f16", 8, "structured", False),
    (300, 768, 64, 3, 64, "f16", 129, "structured", False),
    (160, 512, 16, 4, 32, "bf16", 40, "irregular", False),
    (128, 384, 32, 4, 64, "bf16", 70, "structured", True),
]


@pytest.mark.parametrize("case", CASES)
def test_qeftlinear_autograd(Q, case):
    import torch
    from paper_2410_08661_b200.qlinear import QEFTLinear, _weak_columns
    oc, ic, k, bits, g, dt, T, layout, perm = case
    rng = np.random.default_rng(oc * 7 + T)
    w = (rng.standard_normal((oc, ic)) * 0.05).astype(np.float32)
    kw = {"lam": np.abs(rng.standard_normal(ic))} if layout == "irregular" else {}
    q = Q.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn", layout=layout, **kw)
    if perm:
        q.input_perm = rng.permutation(ic).astype(np.int64)
    lin = QEFTLinear.from_quantized(q, dtype=dt)
    W = lin.dl.dequant_full().double()
    x = torch.randn(T, ic, device="cuda").to(lin.dl.tdtype).requires_grad_(True)
    y = lin(x)
    ref = x.detach().double() @ W.T
    assert rel_err(y.detach().float().cpu().numpy(), ref.cpu().numpy()) <= 1e-2
    dy = torch.randn(T, oc, device="cuda").to(lin.dl.tdtype)
    y.backward(dy)
    dx_ref = dy.double() @ W
    assert rel_err(x.grad.float().cpu().numpy(), dx_ref.cpu().numpy()) <= 1e-2
    cols = _weak_columns(lin.dl)
    dw_ref = dy.double().T @ x.detach().double()[:, cols]
    assert rel_err(lin.weak32.grad.cpu().numpy(), dw_ref.cpu().numpy()) <= 1e-2
    # a second micro-batch accumulates into the same .grad (tuning.py:219-224)
    y2 = lin(x.detach())
    y2.backward(dy)
    assert rel_err(lin.weak32.grad.cpu().numpy(), 2 * dw_ref.cpu().numpy()) <= 1e-2
