"""apply_to_device (SURVEY 8(f) #4 on the B200 path): a delta added into a loaded decoder's fp32
weak masters (+ refreshed kernel copy) gives exactly the reference's merged weak blocks
(apply_to_quantized, merging.py:171: the same fp32 add), and the same logits as a decoder
built from the host-merged model. (The merge is base + f32(tuned - base), which need not round
back to the tuned weights bit for bit, in the reference either.)"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("reo", ["ogr", "online"])
def test_apply_to_device_equals_reference_merge(reo):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import container as C
    from paper_2410_08661_b200 import merging as Mg
    base_q = C.load_checkpoint(os.path.join(GOLD, f"toy_{reo}.qeft"))
    delta = C.load_checkpoint(os.path.join(GOLD, f"toy_{reo}.delta.qeft"))
    model = C.load_to_device(os.path.join(GOLD, f"toy_{reo}.qeft"), act_dtype="f16", compute_dtype="f32")
    from paper_2410_08661_b200.model import QEFTDecoder
    from tests.conftest import load_golden
    z = load_golden("container")
    Mg.apply_to_device(model, base_q, delta)
    for (name, _), lin in zip(base_q.layer_items(), model.linears()):
        assert np.array_equal(lin.weak32.detach().cpu().numpy(), z[f"{reo}_merged_{name}"]), name
    host = QEFTDecoder.from_quantized_model(Mg.apply_to_quantized(base_q, delta), act_dtype="f16",
                                            compute_dtype="f32")
    for a, b in zip(model.linears(), host.linears()):
        assert torch.equal(a.dl.weak16, b.dl.weak16)
    tok = torch.randint(0, model.cfg.vocab_size, (2, 20), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    with torch.no_grad():
        assert torch.equal(model(tok), host(tok))
