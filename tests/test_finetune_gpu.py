"""GPU parity of the fine-tuning path against the REFERENCE itself
(tests/golden/finetune.npz, written by tests/golden/make_golden.py from
pkg/src/qeft): the toy decoder (reference SMALL_CONFIG shape) quantized with
OGR and with online reordering, then
  * one forward/backward through QEFTDecoder vs the reference engine with
    QuantLinearTrainOp (model.py:323-479, tuning.py:106-131): logits, loss and
    every layer's dW_weak;
  * three `finetune` steps (tuning.py:187-248): per-step loss and pre-clip
    gradient norm, cost counters (exact) and the final weak blocks.
Tolerances (north_star: <= 1e-2 max-rel vs fp32 reference accumulation):
  logits / loss        max|d| / max(1, max|ref|) <= 1e-2
  dW_weak, weak blocks max|d| / max|ref|        <= 2e-2 (fp16 kernel operands)
"""

import numpy as np
import pytest

from tests.conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu


def _qmodel(z, mi):
    from paper_2410_08661_b200.qmodel import ModelConfig, QuantBlock, QuantizedModel, BLOCK_LINEARS
    from paper_2410_08661_b200.quantizer import QuantizedLinear
    c = [int(v) for v in z["cfg"]]
    cfg = ModelConfig(*c)
    pre = f"m{mi}_"
    blocks = []
    for i in range(cfg.n_blocks):
        layers = {}
        for nm in BLOCK_LINEARS:
            p = f"{pre}b{i}.{nm}_"
            perm = z[p + "input_perm"]
            layers[nm] = QuantizedLinear(
                oc=int(z[p + "oc"]), ic=int(z[p + "ic"]), k=int(z[p + "k"]), bits=int(z[p + "bits"]),
                g=int(z[p + "g"]), packed=z[p + "packed"].tobytes(), scales=z[p + "scales"],
                zeros=z[p + "zeros"], weak=z[p + "weak"].copy(), weak_indices=z[p + "weak_indices"],
                layout=str(z[p + "layout"]), mode="rtn",
                input_perm=perm if perm.size else None)
        blocks.append(QuantBlock(gain1=z[f"{pre}b{i}_gain1"], gain2=z[f"{pre}b{i}_gain2"], layers=layers))
    return QuantizedModel(config=cfg, embedding=z[pre + "embedding"], blocks=blocks,
                          final_gain=z[pre + "final_gain"], head=z[pre + "head"])


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


@pytest.fixture(scope="module")
def Z():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return load_golden("finetune")


@pytest.mark.parametrize("mi,cdt", [(0, "f32"), (1, "f32"), (0, "f16"), (1, "f16")])
def test_forward_backward_vs_reference_engine(Z, mi, cdt):
    import torch
    from paper_2410_08661_b200.model import QEFTDecoder, cross_entropy_mean
    qm = _qmodel(Z, mi)
    model = QEFTDecoder.from_quantized_model(qm, act_dtype="f16", compute_dtype=cdt)
    xb = torch.from_numpy(Z[f"m{mi}_xb"]).cuda()
    yb = torch.from_numpy(Z[f"m{mi}_yb"]).cuda()
    logits = model(xb)
    loss = cross_entropy_mean(logits, yb)
    scale = 64.0  # exact loss scale for the fp16 kernels, divided back out below
    (loss * scale).backward()
    ref_logits = Z[f"m{mi}_logits"].transpose(0, 2, 1)  # reference (B, V, T)
    assert rel_err(logits.detach().float().cpu().numpy(), ref_logits) <= 1e-2
    assert abs(float(loss.detach()) - float(Z[f"m{mi}_loss"])) <= 1e-2 * max(1.0, abs(float(Z[f"m{mi}_loss"])))
    worst = 0.0
    for lin in model.linears():
        ref = Z[f"m{mi}_grad_{lin.name}"]
        got = lin.weak32.grad.cpu().numpy() / scale
        worst = max(worst, _rel(got, ref))
    print(f"model {mi}: worst dW_weak rel {worst:.3e}")
    assert worst <= 2e-2


@pytest.mark.parametrize("mi,cdt", [(0, "f32"), (1, "f32"), (0, "f16"), (1, "f16")])
def test_finetune_three_steps_vs_reference(Z, mi, cdt):
    """compute_dtype f16 is the precision bench.py's 7B fine-tune step runs at (fp16 kernels,
    fp16 residual stream, exact power-of-two loss scale)."""
    from paper_2410_08661_b200.tuning import TuneConfig, finetune
    qm = _qmodel(Z, mi)
    ids = Z["ids"]
    tc = TuneConfig(steps=3, lr=1e-3, batch=2, grad_accum=2, seq_len=32, seed=2, log_every=1)
    tuned, log = finetune(qm, ids, tc, act_dtype="f16", compute_dtype=cdt)
    loss = np.array([r["loss"] for r in log])
    gnorm = np.array([r["grad_norm"] for r in log])
    counts = np.array([[r["wgrad_fma"], r["full_fma"], r["saved_elems"], r["full_elems"]] for r in log])
    np.testing.assert_array_equal(counts, Z[f"m{mi}_log_counts"])
    assert rel_err(loss, Z[f"m{mi}_log_loss"]) <= 1e-2
    assert _rel(gnorm, Z[f"m{mi}_log_gnorm"]) <= 2e-2
    worst = 0.0
    for name, q in tuned.layer_items():
        worst = max(worst, _rel(q.weak, Z[f"m{mi}_tuned_{name}"]))
    print(f"model {mi}: loss {loss} ref {Z[f'm{mi}_log_loss']}; worst weak rel {worst:.3e}")
    assert worst <= 2e-2
    # frozen parts untouched (pkg/tests/test_tuning.py:193-205)
    ref_qm = _qmodel(Z, mi)
    for (n, q1), (_, q2) in zip(ref_qm.layer_items(), tuned.layer_items()):
        assert q1.packed == q2.packed and np.array_equal(q1.scales, q2.scales)
