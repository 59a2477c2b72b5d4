"""7B-shaped QEFT fine-tune step on one GPU: build the synthetic model, run
warm-up + timed steps (CUDA events), print tokens/s and a phase breakdown."""
import os, sys, time, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.qmodel import LLAMA2_7B, ModelConfig
from paper_2410_08661_b200.model import QEFTDecoder, cross_entropy_mean
from paper_2410_08661_b200.tuning import TuneConfig, WeakTrainer

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=32)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--mb", type=int, default=1)
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
cfg = ModelConfig(**{**LLAMA2_7B.__dict__, "n_blocks": args.blocks})
t0 = time.time()
model = QEFTDecoder.synthetic(cfg, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
tr = WeakTrainer(model, TuneConfig(lr=5e-6, max_grad_norm=0.3))
torch.cuda.synchronize()
print("build s", round(time.time() - t0, 1), "weak params", tr.n_params, "mem GB", round(torch.cuda.memory_allocated() / 1e9, 2), flush=True)
V = cfg.vocab_size
tok = torch.randint(0, V, (args.mb, args.seq + 1), device="cuda")
x, y = tok[:, :-1], tok[:, 1:]
ev = lambda: torch.cuda.Event(enable_timing=True)
def step(times=None):
    e = [ev() for _ in range(4)]
    e[0].record()
    tr.zero_grad()
    loss = cross_entropy_mean(model(x), y)
    e[1].record()
    loss.backward()
    e[2].record()
    tr.step(1)
    e[3].record()
    if times is not None:
        times.append(e)
    return loss
for _ in range(2):
    l = step()
torch.cuda.synchronize()
print("loss", float(l), "peak mem GB", round(torch.cuda.max_memory_allocated() / 1e9, 2), flush=True)
times = []
s0, s1 = ev(), ev()
s0.record()
for _ in range(args.steps):
    step(times)
s1.record()
torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / args.steps
ph = [sum(e[i].elapsed_time(e[i + 1]) for e in times) / len(times) for i in range(3)]
print(json.dumps({"ms_per_step": ms, "tokens_per_s": args.mb * args.seq / ms * 1e3,
                  "fwd_ms": ph[0], "bwd_ms": ph[1], "opt_ms": ph[2], "blocks": args.blocks}))
