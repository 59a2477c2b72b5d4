"""Parity on the BASELINE.json config shapes beyond the 7B decode stack:
  * configs[3]  LLaMA-2-13B-shaped 3-bit layers (d=5120, ff=13824): decode GEMV
    and the prefill / fine-tune GEMMs (fwd, dX, dW_weak) at T = 512;
  * configs[4]  LLaMA-2-70B shapes (8192 x 28672 and 28672 x 8192), 4-bit, weak-column
    ratio sweep k in {16, 32, 64, 128, 256}: m mod 128 = 112 / 96 / 64 / 0 / 0, so the
    ragged last group and the padded tile tail are exercised.
Rows are sliced to a few row-blocks (the kernels' row-blocks are independent), the
K extent is the full model width. Reference: fp64 product over the device-
dequantized weights; tolerance max|d| / max(1, max|ref|) <= 1e-2 (north_star)."""

import numpy as np
import pytest

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import quantizer
    return quantizer


def _layer(Q, oc, ic, k, bits, g=128, seed=0):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((oc, ic)) * 0.02).astype(np.float32)
    return Q.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn")


def _check_all(q, dtype, n_cols, T):
    import torch
    dl = q.device(dtype)
    W = dl.dequant_full().double()
    # decode GEMV
    x = torch.randn(n_cols, q.ic, device="cuda").to(dl.tdtype)
    y = dl.gemv(x, out_f32=True)
    assert rel_err(y.cpu().numpy(), (x.double() @ W.T).cpu().numpy()) <= TOL
    # prefill / fine-tune GEMMs
    X = torch.randn(T, q.ic, device="cuda").to(dl.tdtype)
    dY = torch.randn(T, q.oc, device="cuda").to(dl.tdtype)
    assert rel_err(dl.gemm_fwd(X).float().cpu().numpy(), (X.double() @ W.T).cpu().numpy()) <= TOL
    assert rel_err(dl.gemm_dgrad(dY).float().cpu().numpy(), (dY.double() @ W).cpu().numpy()) <= TOL
    wc = torch.from_numpy(np.asarray(q.weak_indices)).cuda()
    xw = dl.gather_weak(X)
    dw = dl.gemm_wgrad_weak(dY, xw)
    assert rel_err(dw.cpu().numpy(), (dY.double().T @ X.double()[:, wc]).cpu().numpy()) <= TOL


@pytest.mark.parametrize("oc,ic", [(64, 5120), (64, 13824), (48, 5120)])
def test_13b_3bit_shapes(Q, oc, ic):
    q = _layer(Q, oc, ic, k=128, bits=3, seed=oc + ic)
    _check_all(q, "bf16", n_cols=4, T=512)


@pytest.mark.parametrize("k", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("oc,ic", [(48, 8192), (32, 28672)])
def test_70b_weak_ratio_sweep(Q, oc, ic, k):
    q = _layer(Q, oc, ic, k=k, bits=4, seed=k + ic)
    assert (q.m % 128) == {16: 112, 32: 96, 64: 64, 128: 0, 256: 0}[k]
    _check_all(q, "f16", n_cols=1, T=256)
