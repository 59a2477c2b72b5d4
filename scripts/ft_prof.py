"""Kernel-time breakdown of the fine-tune step (torch.profiler / CUPTI)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2410_08661_b200.qmodel import LLAMA2_7B, ModelConfig
from paper_2410_08661_b200.model import QEFTDecoder, cross_entropy_mean
from paper_2410_08661_b200.tuning import TuneConfig, WeakTrainer
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = ModelConfig(**{**LLAMA2_7B.__dict__, "n_blocks": nb})
model = QEFTDecoder.synthetic(cfg, act_dtype="bf16", compute_dtype="bf16")
tr = WeakTrainer(model, TuneConfig(lr=5e-6))
tok = torch.randint(0, cfg.vocab_size, (1, 2049), device="cuda")
def step():
    tr.zero_grad()
    cross_entropy_mean(model(tok[:, :-1]), tok[:, 1:]).backward()
    tr.step(1)
for _ in range(2): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2): step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=90))
