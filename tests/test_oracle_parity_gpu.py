"""Every product entry point pinned to the CPU oracle (oracle/qeft_oracle.py, itself pinned to
the reference's golden vectors by tests/test_oracle_golden.py):

  * the device dequant (`qeft_dequant_full`) vs O.dequant_full, element for element;
  * the product's numpy-facing reference names -- tuning.qlinear_forward_train /
    qlinear_backward, QuantLinearTrainOp, qmodel.QuantLinearInferOp, kernels.KernelPathOp,
    matvec_dispatch (every path incl. "reference") -- on the reference's own training
    fixtures (tests/golden/training.npz, written by pkg/src/qeft/tuning.py:52-103);
  * the drop-in contract with the reference's OWN record shape: OracleLayer records (the
    reference's QuantizedLinear fields, quantizer.py:42-57, no `.device`) through
    QuantLinearTrainOp with the weak block updated IN PLACE between steps as the reference
    fine-tune loop does (tuning.py:148-160, 234-236);
  * SURVEY 8(d) Cfg1 (4096x4096, 4-bit, g128, k=128) forward + dX + dW_weak at T = 1 and
    T = 2048 vs O.forward_train / O.backward (configs[0] is fwd+bwd at batch 1).

Tolerance (north_star): max|y - ref| / max(1, max|ref|) <= 1e-2 (pkg/tests/test_kernels.py:37
metric) against the oracle's fp32/fp64 accumulation; integer outputs (saved x_weak slice,
counters) exact."""

import copy

import numpy as np
import pytest

from oracle import qeft_oracle as O
from tests.conftest import golden_layer, load_golden, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import kernels, qmodel, quantizer, tuning
    return kernels, qmodel, quantizer, tuning


def _oracle_record(q):
    """Any record with the reference fields -> the oracle's own record class."""
    return O.OracleLayer(oc=q.oc, ic=q.ic, k=q.k, bits=q.bits, g=q.g, packed=bytes(q.packed),
                         scales=np.asarray(q.scales), zeros=np.asarray(q.zeros),
                         weak=np.array(q.weak, np.float32), weak_indices=np.asarray(q.weak_indices),
                         layout=q.layout, input_perm=q.input_perm)


def _golden_record(z, t):
    q = golden_layer(z, f"t{t}_")
    perm = z[f"t{t}_input_perm"]
    q.input_perm = perm if perm.size else None
    return q


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", [
    # oc, ic, k, bits, g, layout, online
    (64, 1024, 128, 4, 128, "structured", False),
    (48, 1100, 12, 3, 128, "structured", False),     # ragged last group, 3-bit
    (40, 520, 16, 4, 32, "irregular", False),
    (33, 384, 32, 4, 64, "structured", True),         # online input permutation
    (17, 200, 8, 3, 40, "structured", False),          # g not a multiple of 64
])
def test_device_dequant_vs_oracle(P, case):
    from paper_2410_08661_b200.layer import device_layer
    _, _, quantizer, _ = P
    oc, ic, k, bits, g, layout, online = case
    rng = np.random.default_rng(oc * ic)
    w = (rng.standard_normal((oc, ic)) * 0.05).astype(np.float32)
    kw = {"lam": np.abs(rng.standard_normal(ic))} if layout == "irregular" else {}
    q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn", layout=layout, **kw)
    if online:
        q.input_perm = rng.permutation(ic).astype(np.int64)
    o = _oracle_record(q)
    ref = o.dequant_full()                       # reordered-channel coordinates
    if online:                                   # device dequant is in ORIGINAL coordinates
        full = np.empty_like(ref)
        full[:, o.input_perm] = ref
        ref = full
    got = device_layer(q, "f16").dequant_full().cpu().numpy()
    qcols = o.quant_positions() if not online else o.input_perm[o.quant_positions()]
    wcols = o.weak_indices if not online else o.input_perm[o.weak_indices]
    # quantized columns: f32(c)*s + z with one rounding (FMA) instead of two (mul, then add):
    # at most one ulp of the row's largest term apart
    dq = np.abs(got[:, qcols] - ref[:, qcols])
    row_scale = np.abs(ref[:, qcols]).max(axis=1, keepdims=True) + np.abs(o.zeros).max(axis=1, keepdims=True)
    assert np.all(dq <= 2.0 ** -22 * row_scale)
    # weak columns: the fp16 kernel shadow of the fp32 master
    assert np.array_equal(got[:, wcols], ref[:, wcols].astype(np.float16).astype(np.float32))


# ---------------------------------------------------------------------------
def test_product_train_names_vs_reference_fixtures(P):
    """tuning.qlinear_forward_train / qlinear_backward on reference-shaped records vs the
    reference's own outputs (training.npz), plus the oracle at the same inputs."""
    _, _, _, tuning = P
    z = load_golden("training")
    for t in range(int(z["n"])):
        q = _golden_record(z, t)
        x, dy = z[f"t{t}_x"], z[f"t{t}_dy"]
        y, st = tuning.qlinear_forward_train(q, x)
        assert rel_err(y, z[f"t{t}_y"]) <= TOL, t
        assert np.array_equal(st.x_weak, z[f"t{t}_xw"]), t
        c = tuning.CostCounters()
        dx, dw = tuning.qlinear_backward(st, dy, q, counters=c)
        assert rel_err(dx, z[f"t{t}_dx"]) <= TOL, t
        assert rel_err(dw, z[f"t{t}_dw"]) <= TOL, t
        assert [c.wgrad_fma, c.full_fma, c.saved_elems, c.full_elems] == list(z[f"t{t}_counters"]), t
        y_o, xw_o = O.forward_train(q, x)
        assert rel_err(y, y_o) <= TOL and np.array_equal(st.x_weak, xw_o)


def test_protocol_ops_vs_reference_fixtures(P):
    """QuantLinearTrainOp, QuantLinearInferOp and KernelPathOp (model.py:192-216 protocol)
    on the reference's fixtures: apply / forward_train / backward."""
    kernels, qmodel, _, tuning = P
    z = load_golden("training")
    for t in range(int(z["n"])):
        q = _golden_record(z, t)
        x, dy = z[f"t{t}_x"], z[f"t{t}_dy"]
        op = tuning.QuantLinearTrainOp(f"l{t}", q)
        assert op.always_weight_grad and (op.oc, op.ic) == (q.oc, q.ic)
        y, st = op.forward_train(x)
        dx, dw = op.backward(st, dy, True)
        assert rel_err(y, z[f"t{t}_y"]) <= TOL and rel_err(op.apply(x), z[f"t{t}_y"]) <= TOL
        assert rel_err(dx, z[f"t{t}_dx"]) <= TOL and rel_err(dw, z[f"t{t}_dw"]) <= TOL
        inf = qmodel.QuantLinearInferOp(f"l{t}", q)
        yi, sti = inf.forward_train(x)
        assert sti is None and rel_err(yi, z[f"t{t}_y"]) <= TOL
        dxi, dwi = inf.backward(sti, dy, True)
        assert dwi is None and rel_err(dxi, z[f"t{t}_dx"]) <= TOL
        # the kernel-path op runs matvec_dispatch per column (kernels.py:163-186): the native
        # path, whose online-reorder form takes x[perm[:m]] / x[perm[m:]] whatever the layout
        # (kernels.py:115-126) -- for the fixture's irregular + input_perm layer that differs
        # from the training product, exactly as in the reference
        stats = {}
        kp = kernels.KernelPathOp(f"l{t}", q, stats)
        ref_native = np.stack([O.matvec_native(q, x[:, j]) for j in range(x.shape[1])], axis=1)
        assert rel_err(kp.apply(x), ref_native) <= TOL, t
        assert stats[f"l{t}"].calls == x.shape[1]
        kr = kernels.KernelPathOp(f"l{t}", q, {}, reference=True)
        ref_dense = np.stack([O.matvec_reference(q, x[:, j]) for j in range(x.shape[1])], axis=1)
        assert rel_err(kr.apply(x), ref_dense) <= TOL, t


def test_matvec_every_path_vs_oracle(P):
    """matvec_dispatch over the native path vs O.matvec_native, and the dense 'reference' path
    (online layers included: the device dequant is already in original coordinates, so x is
    not permuted a second time) vs O.matvec_reference."""
    kernels, _, _, _ = P
    z = load_golden("training")
    for t in range(int(z["n"])):
        q = _golden_record(z, t)
        x = z[f"t{t}_x"][:, 0]
        assert rel_err(kernels.matvec_dispatch(q, x), O.matvec_native(q, x)) <= TOL, t
        assert rel_err(kernels.matvec_dispatch(q, x, path="reference"), O.matvec_reference(q, x)) <= TOL, t


def test_fp32_inputs_beyond_fp16_range(P):
    """x with |x| > 65504 goes through the fp16 kernels via an exact power-of-two scale."""
    kernels, _, quantizer, tuning = P
    rng = np.random.default_rng(3)
    w = (rng.standard_normal((48, 256)) * 0.05).astype(np.float32)
    q = quantizer.quantize_layer(w, k=16, bits=4, g=64, mode="rtn")
    x = (rng.standard_normal(256) * 3e5).astype(np.float32)
    ref = O.matvec_native(_oracle_record(q), x)
    y = kernels.matvec_structured(q, x)
    assert np.all(np.isfinite(y)) and rel_err(y, ref) <= TOL
    X = (rng.standard_normal((256, 40)) * 3e5).astype(np.float32)
    yt, _ = tuning.qlinear_forward_train(q, X)
    assert rel_err(yt, O.forward_train(_oracle_record(q), X)[0]) <= TOL


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("t", [0, 1, 3, 5])
def test_reference_records_inplace_adam_loop(P, t):
    """The reference fine-tune loop, per layer: forward_train -> backward -> adam_step IN PLACE
    on q.weak, 3 steps, on records of the reference's own shape (no .device). Each forward must
    see the updated weak block: a stale device copy is caught by the step-2/3 comparisons."""
    _, _, _, tuning = P
    z = load_golden("training")
    q = _golden_record(z, t)          # product op state
    o = copy.deepcopy(q)              # oracle twin
    assert not hasattr(q, "device")
    rng = np.random.default_rng(40 + t)
    op = tuning.QuantLinearTrainOp("l", q)
    st_p = O.AdamMoments(m=np.zeros_like(q.weak), v=np.zeros_like(q.weak))
    st_o = O.AdamMoments(m=np.zeros_like(o.weak), v=np.zeros_like(o.weak))
    w0 = q.weak.copy()
    for step in range(3):
        x = rng.standard_normal((q.ic, 9)).astype(np.float32)
        dy = rng.standard_normal((q.oc, 9)).astype(np.float32)
        y, st = op.forward_train(x)
        y_o, xw_o = O.forward_train(o, x)
        assert rel_err(y, y_o) <= TOL, step
        if step:
            stale = _oracle_record(q)
            stale.weak = w0
            # the update is large enough that a stale weak block would fail the bar
            assert rel_err(O.forward_train(stale, x)[0], y_o) > 2 * TOL
        dx, dw = op.backward(st, dy, True)
        dx_o, dw_o = O.backward(o, xw_o, dy)
        assert rel_err(dx, dx_o) <= TOL and rel_err(dw, dw_o) <= TOL
        O.adam_update(st_p, q.weak, dw, lr=0.5)     # in place, like tuning.adam_step
        O.adam_update(st_o, o.weak, dw_o, lr=0.5)
    assert rel_err(q.weak, o.weak) <= 2e-2


# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def cfg1(P):
    """W ~ N(0, 0.02^2) seed 0, lambda-selected weak block moved to the tail,
    quantize_layer(k=128, bits=4, g=128, rtn, structured)."""
    from paper_2410_08661_b200 import calibration, reorder
    _, _, quantizer, _ = P
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((4096, 4096)) * 0.02).astype(np.float32)
    r1 = np.random.default_rng(1)
    xc = r1.standard_normal((4096, 256)).astype(np.float32)
    xc[r1.choice(4096, 128, replace=False)] *= 10
    lam = 2.0 * np.sum(xc.astype(np.float64) ** 2, axis=1)
    perm = reorder.weak_to_tail(4096, calibration.select_local_topk(lam, 128))
    q = quantizer.quantize_layer(perm.apply_cols(w), k=128, bits=4, g=128, mode="rtn")
    return q, _oracle_record(q)


@pytest.mark.parametrize("T", [1, 2048])
def test_cfg1_fwd_bwd_vs_oracle(P, cfg1, T):
    _, _, _, tuning = P
    q, o = cfg1
    rng = np.random.default_rng(3)
    x = rng.standard_normal((4096, T)).astype(np.float32)
    dy = np.random.default_rng(4).standard_normal((4096, T)).astype(np.float32)
    y, st = tuning.qlinear_forward_train(q, x)
    y_o, xw_o = O.forward_train(o, x)
    assert rel_err(y, y_o) <= TOL
    assert np.array_equal(st.x_weak, xw_o)
    dx, dw = tuning.qlinear_backward(st, dy, q)
    dx_o, dw_o = O.backward(o, xw_o, dy)
    e = (rel_err(dx, dx_o), rel_err(dw, dw_o))
    print(f"Cfg1 T={T}: fwd {rel_err(y, y_o):.2e} dX {e[0]:.2e} dW {e[1]:.2e}")
    assert max(e) <= TOL
