"""7B-shaped end-to-end decode step (KVDecoder, CUDA graph, batch 1): ms/token at a given
context length, for the bench's decode_step sub-object."""
import os, sys, time, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.qmodel import LLAMA2_7B, ModelConfig
from paper_2410_08661_b200.model import QEFTDecoder
from paper_2410_08661_b200.generate import KVDecoder

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=32)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--steps", type=int, default=32)
a = ap.parse_args()
cfg = ModelConfig(**{**LLAMA2_7B.__dict__, "n_blocks": a.blocks})
t0 = time.time()
model = QEFTDecoder.synthetic(cfg, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
for p in model.parameters():
    p.requires_grad_(False)
dec = KVDecoder(model, max_seq=a.ctx + a.steps + 1, capture=True)
print("build s", round(time.time() - t0, 1), flush=True)
tok = torch.tensor([1])
for p in range(a.ctx):
    dec.step(tok, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for i in range(a.steps):
    dec.step(tok, a.ctx + i)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(json.dumps({"ms_per_token": ms, "tokens_per_s": 1e3 / ms, "ctx": a.ctx, "blocks": a.blocks}))
