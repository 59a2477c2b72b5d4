"""End-to-end decode around the GEMV: the KV-cache decoder against the
reference's greedy harness bench_generate (pkg/src/qeft/kernels.py:197-228) on the toy
quantized models of tests/golden/toy_*.qeft.
  * every decode step's logits vs column p of the reference's full causal forward over the
    final sequence: max|d| / max(1, max|ref|) <= 1e-2 (fp16 activations), eager and
    CUDA-graph modes;
  * greedy tokens identical to the reference's."""

import os

import numpy as np
import pytest

from tests.conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def Z():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return load_golden("container")


def _model(reo):
    from paper_2410_08661_b200.container import load_to_device
    return load_to_device(os.path.join(GOLD, f"toy_{reo}.qeft"), act_dtype="f16", compute_dtype="f16")


@pytest.mark.parametrize("reo", ["ogr", "online"])
@pytest.mark.parametrize("capture", [False, True])
def test_decode_steps_match_full_forward(Z, reo, capture):
    import torch
    from paper_2410_08661_b200.generate import KVDecoder
    dec = KVDecoder(_model(reo), capture=capture)
    seq = np.concatenate([Z[f"{reo}_prompt"], Z[f"{reo}_gen_tokens"]])[:-1]
    ref = Z[f"{reo}_gen_logits"][0]  # (V, T)
    worst = 0.0
    for p, t in enumerate(seq):
        lg = dec.step(torch.tensor([int(t)]), p)[0].cpu().numpy()
        worst = max(worst, rel_err(lg, ref[:, p]))
    assert worst <= 1e-2, worst


@pytest.mark.parametrize("reo", ["ogr", "online"])
def test_greedy_tokens_match_reference(Z, reo):
    from paper_2410_08661_b200.generate import bench_generate
    from paper_2410_08661_b200.container import load_checkpoint
    qm = load_checkpoint(os.path.join(GOLD, f"toy_{reo}.qeft"))
    res = bench_generate(qm, Z[f"{reo}_prompt"], 10, repeats=2)
    assert np.array_equal(res.tokens, Z[f"{reo}_gen_tokens"]), (res.tokens, Z[f"{reo}_gen_tokens"])
    assert res.tokens_per_s > 0


def test_decoder_rejects_bad_positions(Z):
    import torch
    from paper_2410_08661_b200.errors import ShapeError
    from paper_2410_08661_b200.generate import KVDecoder, generate
    dec = KVDecoder(_model("ogr"), max_seq=16)
    with pytest.raises(ShapeError):
        dec.step(torch.tensor([1]), 16)
    with pytest.raises(ShapeError):
        generate(dec, np.arange(10), 10)
