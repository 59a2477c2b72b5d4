"""torch.profiler view of one 7B fine-tune step (4 blocks): which aten ops launch the copy /
add kernels, with Python call sites."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2410_08661_b200.qmodel import LLAMA2_7B, ModelConfig
from paper_2410_08661_b200.model import QEFTDecoder, cross_entropy_mean
from paper_2410_08661_b200.tuning import TuneConfig, WeakTrainer
cfg = ModelConfig(**{**LLAMA2_7B.__dict__, "n_blocks": 4})
model = QEFTDecoder.synthetic(cfg, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
tr = WeakTrainer(model, TuneConfig(lr=5e-6, max_grad_norm=0.3))
tok = torch.randint(0, cfg.vocab_size, (1, 2049), device="cuda")
x, y = tok[:, :-1], tok[:, 1:]
def step():
    tr.zero_grad()
    loss = cross_entropy_mean(model(x), y)
    loss.backward()
    tr.step(1)
for _ in range(2): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as p:
    step(); torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(p.key_averages(group_by_stack_n=6).table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=50))
