"""Parity on the BASELINE.json config shapes beyond the 7B decode stack:
  * configs[3]  LLaMA-2-13B-shaped 3-bit layers (d=5120, ff=13824): decode GEMV
    and the prefill / fine-tune GEMMs (fwd, dX, dW_weak) at T = 512;
  * configs[4]  LLaMA-2-70B shapes (8192 x 28672 and 28672 x 8192), 4-bit, weak-column
    ratio sweep k in {16, 32, 64, 128, 256}: m mod 128 = 112 / 96 / 64 / 0 / 0, so the
    ragged last group and the padded tile tail are exercised.
Rows are sliced to a few row-blocks (the kernels' row-blocks are independent), the
K extent is the full model width; the 7B shapes (configs[1]/[2]) run at full size.
Reference: the CPU oracle (O.matvec_native / O.forward_train / O.backward, fp64 / fp32
accumulation over the oracle's own dequant of the same record); tolerance
max|d| / max(1, max|ref|) <= 1e-2 (north_star)."""

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


def _f16_exact(a, dtype):
    """Host fp32 values exactly representable in the kernel operand dtype."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(
        torch.float16 if dtype == "f16" else torch.bfloat16)
    return t.float().numpy(), t


def _check_all(q, dtype, n_cols, T):
    from oracle import qeft_oracle as O
    o = O.OracleLayer(oc=q.oc, ic=q.ic, k=q.k, bits=q.bits, g=q.g, packed=bytes(q.packed),
                      scales=q.scales, zeros=q.zeros, weak=q.weak, weak_indices=q.weak_indices,
                      layout=q.layout)
    dl = q.device(dtype)
    rng = np.random.default_rng(q.oc + q.ic + q.k)
    # weak block as the kernels hold it (fp16/bf16 shadow of the fp32 master)
    o.weak = _f16_exact(q.weak, dtype)[0]
    # decode GEMV
    xh, xt = _f16_exact(rng.standard_normal((n_cols, q.ic)), dtype)
    y = dl.gemv(xt.cuda(), out_f32=True).cpu().numpy()
    ref = np.stack([O.matvec_native(o, xh[j]) for j in range(n_cols)])
    assert rel_err(y, ref) <= TOL
    # prefill / fine-tune GEMMs
    Xh, Xt = _f16_exact(rng.standard_normal((T, q.ic)), dtype)
    dYh, dYt = _f16_exact(rng.standard_normal((T, q.oc)), dtype)
    y_o, xw_o = O.forward_train(o, Xh.T)
    dx_o, dw_o = O.backward(o, xw_o, dYh.T)
    Xt, dYt = Xt.cuda(), dYt.cuda()
    assert rel_err(dl.gemm_fwd(Xt).float().cpu().numpy(), y_o.T) <= TOL
    assert rel_err(dl.gemm_dgrad(dYt).float().cpu().numpy(), dx_o.T) <= TOL
    dw = dl.gemm_wgrad_weak(dYt, dl.gather_weak(Xt)).cpu().numpy()
    assert rel_err(dw, dw_o) <= TOL


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


@pytest.mark.parametrize("oc,ic", [(11008, 4096), (4096, 11008)])
def test_7b_full_shapes(Q, oc, ic):
    """configs[1]/[2] shapes at full size (gate/up and down), 4-bit g128 k=128."""
    q = _layer(Q, oc, ic, k=128, bits=4, seed=oc)
    _check_all(q, "f16", n_cols=1, T=256)
