"""Kernel time breakdown of the 7B decode step (CUDA-graph replay, ctx 512) via torch.profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2410_08661_b200.qmodel import LLAMA2_7B
from paper_2410_08661_b200.model import QEFTDecoder
from paper_2410_08661_b200.generate import KVDecoder
model = QEFTDecoder.synthetic(LLAMA2_7B, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
for p in model.parameters(): p.requires_grad_(False)
dec = KVDecoder(model, max_seq=545, capture=True)
tok = torch.tensor([1])
for p in range(512): dec.step(tok, p)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(4): dec.step(tok, 512 + i)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20, max_name_column_width=90))
