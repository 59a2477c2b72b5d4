"""GPU parity of the tcgen05 GEMMs (fwd, dgrad, wgrad) against the CPU oracle
(reference golden vectors, tuning.py:52-103) and an fp64 product over the
device-dequantized weights. Tolerance: max-rel 1e-2 (BASELINE.json north_star),
metric max|y-ref| / max(1, max|ref|)."""

import numpy as np
import pytest

from oracle import qeft_oracle as O
from tests.conftest import golden_layer, load_golden, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import quantizer
    return quantizer


def _layer(quantizer, oc, ic, k, bits, g, layout="structured", seed=0, perm=False):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((oc, ic)) * 0.05).astype(np.float32)
    kw = {}
    if layout == "irregular":
        kw["lam"] = np.abs(rng.standard_normal(ic))
    q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn", layout=layout, **kw)
    if perm:
        q.input_perm = rng.permutation(ic).astype(np.int64)
    return q


CASES = [
    # oc, ic, k, bits, g, dtype, T, layout, perm
    (512, 1024, 128, 4, 128, "bf16", 256, "structured", False),
    (512, 1024, 128, 4, 128, "f16", 100, "structured", False),
    (4096, 4096, 128, 4, 128, "bf16", 512, "structured", False),
    (300, 2176, 64, 4, 64, "f16", 300, "structured", False),
    (200, 1100, 12, 3, 128, "bf16", 33, "structured", False),
    (256, 768, 64, 3, 128, "bf16", 130, "structured", False),
    (160, 512, 16, 4, 32, "bf16", 64, "irregular", False),
    (128, 384, 32, 4, 64, "bf16", 200, "structured", True),
    (96, 200, 8, 4, 40, "f16", 17, "structured", False),
    # T > 256: two 256-token sub-tiles share each dequantized A stage (ragged last tile)
    (256, 768, 64, 3, 128, "bf16", 700, "structured", False),
    (160, 512, 16, 4, 32, "f16", 520, "irregular", False),
    (128, 384, 32, 4, 64, "bf16", 1000, "structured", True),
    # 20 m-blocks x 8 token pairs = 160 tiles > 148 SMs: the tail wave runs as half tiles
    (2560, 512, 64, 4, 128, "bf16", 4000, "structured", False),
    (512, 2560, 64, 4, 128, "f16", 4000, "structured", False),
    # k % 4 != 0: scalar wgrad epilogue; 1 channel block -> 8-CTA wgrad cluster
    (96, 200, 6, 4, 40, "bf16", 600, "structured", False),
]


@pytest.mark.parametrize("case", CASES)
def test_fwd_dgrad_wgrad_vs_fp64(Q, case):
    import torch
    oc, ic, k, bits, g, dt, T, layout, perm = case
    q = _layer(Q, oc, ic, k, bits, g, layout, seed=oc + ic, perm=perm)
    dl = q.device(dt)
    # W_hat placed at the ORIGINAL input columns: online-reorder layers read x[input_perm]
    # (tuning.py:64-65) and un-permute dX (tuning.py:93-96), which this absorbs
    dq = dl.dequant_full().double()
    x = torch.randn(T, ic, device="cuda").to(dl.tdtype)
    dy = torch.randn(T, oc, device="cuda").to(dl.tdtype)
    y = dl.gemm_fwd(x)
    ref = x.double() @ dq.T
    assert rel_err(y.float().cpu().numpy(), ref.cpu().numpy()) <= TOL
    dx = dl.gemm_dgrad(dy)
    dref = dy.double() @ dq
    assert rel_err(dx.float().cpu().numpy(), dref.cpu().numpy()) <= TOL
    # wgrad on the weak columns x[:, P[weak_indices]]
    p = q.input_perm if perm else np.arange(ic)
    widx = torch.from_numpy(p[q.weak_indices]).cuda()
    dw = dl.gemm_wgrad(dy, x)
    wref = dy.double().T @ x[:, widx].double()
    assert rel_err(dw.cpu().numpy(), wref.cpu().numpy()) <= TOL
    # accumulate paths
    dw2 = dl.gemm_wgrad(dy, x, out=dw.clone(), accumulate=True)
    assert rel_err(dw2.cpu().numpy(), 2 * wref.cpu().numpy()) <= TOL
    dx2 = dl.gemm_dgrad(dy, out=dx.clone(), accumulate=True)
    assert rel_err(dx2.float().cpu().numpy(), 2 * dref.cpu().numpy()) <= TOL


def test_train_golden_vs_reference(Q):
    """Reference qlinear_forward_train / qlinear_backward golden vectors
    (tests/golden/training.npz, made by pkg/src/qeft/tuning.py)."""
    import torch
    z = load_golden("training")
    for t in range(int(z["n"])):
        p = f"t{t}_"
        o = golden_layer(z, p)
        ip = z[p + "input_perm"]
        q = Q.QuantizedLinear(oc=o.oc, ic=o.ic, k=o.k, bits=o.bits, g=o.g, packed=o.packed,
                              scales=o.scales, zeros=o.zeros, weak=o.weak,
                              weak_indices=o.weak_indices, layout=o.layout,
                              input_perm=ip if ip.size else None)
        dl = q.device("f16")
        x = torch.from_numpy(z[p + "x"].T.copy()).cuda().half()     # (T, ic)
        dy = torch.from_numpy(z[p + "dy"].T.copy()).cuda().half()   # (T, oc)
        y = dl.gemm_fwd(x).float().cpu().numpy().T
        assert rel_err(y, z[p + "y"]) <= TOL, t
        dx = dl.gemm_dgrad(dy).float().cpu().numpy().T
        assert rel_err(dx, z[p + "dx"]) <= TOL, t
        dw = dl.gemm_wgrad(dy, x).cpu().numpy()
        assert rel_err(dw, z[p + "dw"]) <= TOL, t


# stream-K schedule: CTAs own contiguous k-block ranges; a tile split across CTAs is finished
# by the CTA holding its last k-block, which adds the others' fp32 partials. Forced on, small
# layers give every CTA a few k-blocks, so one tile spans many CTAs (multi-producer fix-ups).
def _ulp2(dt):
    """Two output rounding steps of the activation dtype, relative to the largest output."""
    return 2.0 * (2.0 ** -10 if dt == "f16" else 2.0 ** -7)


SK_CASES = [
    (512, 1024, 128, 4, 128, "bf16", 256, "structured", False),   # 4 tiles x 18 k-blocks
    (4096, 4096, 128, 4, 128, "f16", 2048, "structured", False),  # 128 tiles (the 7B shape)
    (4096, 11008, 128, 4, 128, "f16", 2048, "structured", False),  # down_proj
    (11008, 4096, 128, 4, 128, "f16", 2048, "structured", False),  # gate/up: 344 tiles
    (256, 768, 64, 3, 128, "bf16", 700, "structured", False),
    (160, 512, 16, 4, 32, "f16", 520, "irregular", False),
    (128, 384, 32, 4, 64, "bf16", 1000, "structured", True),
    (300, 2176, 64, 4, 64, "f16", 300, "structured", False),
]


SK, PAIRS = 0, 1  # QEFT_SCHED_STREAMK, QEFT_SCHED_CTA_PAIRS


@pytest.fixture
def streamk():
    from paper_2410_08661_b200 import _lib
    L = _lib.lib()
    prev = L.qeft_gemm_set_schedule(SK, 1)
    yield L
    L.qeft_gemm_set_schedule(SK, prev)


@pytest.mark.parametrize("case", SK_CASES)
def test_streamk_matches_whole_tiles(Q, streamk, case):
    import torch
    oc, ic, k, bits, g, dt, T, layout, perm = case
    q = _layer(Q, oc, ic, k, bits, g, layout, seed=oc + ic + 7, perm=perm)
    dl = q.device(dt)
    dq = dl.dequant_full().double()
    x = torch.randn(T, ic, device="cuda").to(dl.tdtype)
    dy = torch.randn(T, oc, device="cuda").to(dl.tdtype)
    y_sk, dx_sk = dl.gemm_fwd(x), dl.gemm_dgrad(dy)
    # deterministic: fixed partition, partials added in CTA order
    assert torch.equal(dl.gemm_fwd(x), y_sk) and torch.equal(dl.gemm_dgrad(dy), dx_sk)
    dx_acc = dl.gemm_dgrad(dy, out=dx_sk.clone(), accumulate=True)
    streamk.qeft_gemm_set_schedule(SK, 0)
    y_dp, dx_dp = dl.gemm_fwd(x), dl.gemm_dgrad(dy)
    streamk.qeft_gemm_set_schedule(SK, 1)
    ref, dref = x.double() @ dq.T, dy.double() @ dq
    assert rel_err(y_sk.float().cpu().numpy(), ref.cpu().numpy()) <= TOL
    assert rel_err(dx_sk.float().cpu().numpy(), dref.cpu().numpy()) <= TOL
    assert rel_err(dx_acc.float().cpu().numpy(), 2 * dref.cpu().numpy()) <= TOL
    # only the fp32 summation order differs from whole tiles: <= 2 output ulps
    ulp2 = _ulp2(dt)
    assert rel_err(y_sk.float().cpu().numpy(), y_dp.float().cpu().numpy()) <= ulp2
    assert rel_err(dx_sk.float().cpu().numpy(), dx_dp.float().cpu().numpy()) <= ulp2


@pytest.mark.parametrize("case", [c for c in CASES if c[6] > 128] + SK_CASES[1:4])
@pytest.mark.parametrize("sk", [0, 1])
def test_cta_pairs_match_single(Q, case, sk):
    """cta_group::2 tiles (M = 256 over two SMs; each CTA dequantizes its own 128 rows and loads
    half of every activation sub-tile; the leader issues the MMAs) against the 1-SM kernel and
    the fp64 product, with whole tiles and with stream-K over CTA pairs."""
    import torch
    from paper_2410_08661_b200 import _lib
    L = _lib.lib()
    oc, ic, k, bits, g, dt, T, layout, perm = case
    q = _layer(Q, oc, ic, k, bits, g, layout, seed=oc + ic + 11, perm=perm)
    dl = q.device(dt)
    dq = dl.dequant_full().double()
    x = torch.randn(T, ic, device="cuda").to(dl.tdtype)
    dy = torch.randn(T, oc, device="cuda").to(dl.tdtype)
    prev_sk = L.qeft_gemm_set_schedule(SK, sk)
    try:
        y1, dx1 = dl.gemm_fwd(x), dl.gemm_dgrad(dy)
        prev = L.qeft_gemm_set_schedule(PAIRS, 2)
        try:
            y2, dx2 = dl.gemm_fwd(x), dl.gemm_dgrad(dy)
            dx2a = dl.gemm_dgrad(dy, out=dx2.clone(), accumulate=True)
        finally:
            L.qeft_gemm_set_schedule(PAIRS, prev)
    finally:
        L.qeft_gemm_set_schedule(SK, prev_sk)
    ref, dref = x.double() @ dq.T, dy.double() @ dq
    assert rel_err(y2.float().cpu().numpy(), ref.cpu().numpy()) <= TOL
    assert rel_err(dx2.float().cpu().numpy(), dref.cpu().numpy()) <= TOL
    assert rel_err(dx2a.float().cpu().numpy(), 2 * dref.cpu().numpy()) <= TOL
    assert rel_err(y2.float().cpu().numpy(), y1.float().cpu().numpy()) <= _ulp2(dt)
    assert rel_err(dx2.float().cpu().numpy(), dx1.float().cpu().numpy()) <= _ulp2(dt)


def test_wgrad_weak_multi_matches_per_layer(Q):
    """qeft_gemm_wgrad_weak_multi (q/k/v-style layers sharing the weak input columns, one launch)
    equals one qeft_gemm_wgrad_weak per layer (the token split may differ: fp32 sums to 1e-5)."""
    import ctypes
    import torch
    from paper_2410_08661_b200 import _lib
    from paper_2410_08661_b200.decode import random_layer
    T = 1000
    dls = [random_layer(oc, 1024, 128, 4, 128, "f16", seed=s) for s, oc in enumerate((512, 384, 512))]
    x = torch.randn(T, 1024, device="cuda").half()
    xw = x[:, dls[0].m:dls[0].m + dls[0].k]
    dys = [torch.randn(T, dl.oc, device="cuda").half() for dl in dls]
    ref = [dl.gemm_wgrad_weak(dy, xw) for dl, dy in zip(dls, dys)]
    out = [torch.full_like(r, 0.5) for r in ref]
    L = _lib.lib()
    n = len(dls)
    arr = (ctypes.POINTER(_lib.QeftLinearT) * n)(*[d.cptr for d in dls])
    dyp = (ctypes.c_void_p * n)(*[d.data_ptr() for d in dys])
    ldd = (ctypes.c_int64 * n)(*[d.stride(0) for d in dys])
    dwp = (ctypes.c_void_p * n)(*[o.data_ptr() for o in out])
    _lib.check(L.qeft_gemm_wgrad_weak_multi(ctypes.cast(arr, ctypes.c_void_p), n, ctypes.cast(dyp, ctypes.c_void_p),
                                            ctypes.cast(ldd, ctypes.c_void_p), xw.data_ptr(), xw.stride(0),
                                            ctypes.cast(dwp, ctypes.c_void_p), T, 1, _lib.stream_ptr()), "multi")
    torch.cuda.synchronize()
    for r, o in zip(ref, out):
        assert rel_err((o - 0.5).cpu().numpy(), r.cpu().numpy()) <= 1e-5
