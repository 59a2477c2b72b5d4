"""Whole-model quantization against the REFERENCE (tests/golden/qmodel.npz, written by
tests/golden/make_golden.py from pkg/src/qeft: qmodel.py:82-156, reorder.py:77-135,
calibration.py:101-187):

  CPU   identity_plan / build_plan / invert_plan / apply_ogr and select_global on the
        reference's own Hessians: permutations, selections and permuted weights bit-exact;
        apply_ogr then the inverted plan restores the model exactly.
  GPU   accumulate_hessian_full over the reference's traced calibration windows (fp64 GEMM on
        the device) vs the reference's Hessians; quantize_model(reorder = ogr | online | none,
        RTN) from those device Hessians vs the reference's quantized models: every record's
        packed codes, scales, zeros, weak block, weak indices, layout and input permutation
        bit-exact, plan / selection / fingerprint identical.
"""

import numpy as np
import pytest

from tests.conftest import load_golden

BL = ("wq", "wk", "wv", "wo", "w_up", "w_gate", "w_down")


@pytest.fixture(scope="module")
def Z():
    return load_golden("qmodel")


def _dense(z):
    from paper_2410_08661_b200.qmodel import DenseBlock, DenseModel, ModelConfig
    cfg = ModelConfig(*[int(v) for v in z["cfg"]])
    blocks = [DenseBlock(**{f: z[f"b{i}_{f}"].copy() for f in ("gain1", "gain2") + BL})
              for i in range(cfg.n_blocks)]
    return DenseModel(config=cfg, embedding=z["embedding"].copy(), blocks=blocks,
                      final_gain=z["final_gain"].copy(), head=z["head"].copy())


def _ref_hess_diag(z):
    from paper_2410_08661_b200.calibration import HessianDiag
    names = [str(n) for n in z["layer_names"]]
    return HessianDiag(lam={n: np.diagonal(z["h_" + n]).copy() for n in names}, sample_count=int(z["n_windows"]))


def test_selection_and_plan_bit_exact(Z):
    from paper_2410_08661_b200 import calibration, reorder
    cfg = _dense(Z).config
    gwc = calibration.select_global(_ref_hess_diag(Z), 4, n_blocks=cfg.n_blocks)
    assert np.array_equal(gwc.resid_indices, Z["gwc_resid"])
    assert np.array_equal(gwc.s_global, Z["gwc_s_global"])
    for i in range(cfg.n_blocks):
        assert np.array_equal(gwc.ffn_indices[i], Z[f"gwc_ffn{i}"])
        assert np.array_equal(gwc.wo_indices[i], Z[f"gwc_wo{i}"])
    plan = reorder.build_plan(gwc, cfg)
    assert np.array_equal(plan.p_resid.perm, Z["plan_resid"])
    for i in range(cfg.n_blocks):
        assert np.array_equal(plan.p_ffn[i].perm, Z[f"plan_ffn{i}"])
    assert not plan.is_identity() and reorder.identity_plan(cfg).is_identity()
    assert len(reorder.identity_plan(cfg).wo_irregular) == cfg.n_blocks


def test_apply_ogr_matches_reference_and_inverts(Z):
    from paper_2410_08661_b200 import reorder
    dense = _dense(Z)
    cfg = dense.config
    plan = reorder.ReorderPlan(p_resid=reorder.Permutation(Z["plan_resid"]),
                               p_ffn=[reorder.Permutation(Z[f"plan_ffn{i}"]) for i in range(cfg.n_blocks)],
                               wo_irregular=[Z[f"gwc_wo{i}"] for i in range(cfg.n_blocks)])
    out = reorder.apply_ogr(dense, plan)
    assert np.array_equal(out.embedding, Z["ogr_embedding"])
    assert np.array_equal(out.head, Z["ogr_head"])
    assert np.array_equal(out.final_gain, Z["ogr_final_gain"])
    for i, b in enumerate(out.blocks):
        assert np.array_equal(b.gain1, Z[f"ogr_b{i}_gain1"]) and np.array_equal(b.gain2, Z[f"ogr_b{i}_gain2"])
        # structured layers: the weak block is the trailing columns of the permuted weight
        for nm in ("wq", "wk", "wv", "w_up", "w_gate", "w_down"):
            k = int(Z[f"ogr_b{i}.{nm}_k"])
            assert np.array_equal(getattr(b, nm)[:, -k:], Z[f"ogr_b{i}.{nm}_weak"]), nm
        # wo: rows permuted, input columns untouched (the irregular weak columns index it)
        assert np.array_equal(b.wo[:, Z[f"ogr_b{i}.wo_weak_indices"]], Z[f"ogr_b{i}.wo_weak"])
    back = reorder.apply_ogr(out, reorder.invert_plan(plan))
    assert np.array_equal(back.embedding, dense.embedding) and np.array_equal(back.head, dense.head)
    for b0, b1 in zip(dense.blocks, back.blocks):
        for f in ("gain1", "gain2") + BL:
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), f
    with pytest.raises(Exception):
        reorder.apply_ogr(dense, reorder.identity_plan(type(cfg)(d_model=16, n_heads=2, head_dim=8, d_ff=64,
                                                                  n_blocks=2)))


@pytest.mark.gpu
def test_accumulate_hessian_full_on_device(Z):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import calibration
    names = [str(n) for n in Z["layer_names"]]
    hf = None
    for w in range(int(Z["n_windows"])):
        acts = {n: torch.from_numpy(Z[f"act{w}_{n}"]).cuda() for n in names}
        hf = calibration.accumulate_hessian_full(acts, hf)
    assert hf.sample_count == int(Z["n_windows"]) and list(hf.h) == names
    for n in names:
        got, ref = hf.h[n].cpu().numpy(), Z["h_" + n]
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), n
    lam = hf.diag().lam
    assert list(lam) == names


@pytest.mark.gpu
@pytest.mark.parametrize("reo", ["ogr", "online", "none"])
def test_quantize_model_bit_exact(Z, reo):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import calibration, qmodel
    names = [str(n) for n in Z["layer_names"]]
    hf = None
    for w in range(int(Z["n_windows"])):
        hf = calibration.accumulate_hessian_full({n: Z[f"act{w}_{n}"] for n in names}, hf)
    qm = qmodel.quantize_model(_dense(Z), hf, k=4, bits=4, g=16, mode="rtn", reorder=reo)
    assert qm.fingerprint == str(Z["fingerprint"]) and qm.reorder == reo
    pre = reo + "_"
    assert np.array_equal(qm.embedding, Z[pre + "embedding"]) and np.array_equal(qm.head, Z[pre + "head"])
    for name, q in qm.layer_items():
        p = pre + name + "_"
        assert q.packed == Z[p + "packed"].tobytes(), name
        for f in ("scales", "zeros", "weak", "weak_indices"):
            assert np.array_equal(getattr(q, f), Z[p + f]), (name, f)
        assert q.layout == str(Z[p + "layout"]) and (q.oc, q.ic, q.k, q.bits, q.g) == tuple(
            int(Z[p + f]) for f in ("oc", "ic", "k", "bits", "g"))
        perm = Z[p + "input_perm"]
        assert (q.input_perm is None) == (perm.size == 0)
        if perm.size:
            assert np.array_equal(q.input_perm, perm)
    if reo == "ogr":
        assert np.array_equal(qm.plan.p_resid.perm, Z["plan_resid"])
        assert np.array_equal(qm.gwc.resid_indices, Z["gwc_resid"])
