"""Probe of the decode-step measurement: the same 7B-shaped KV decode step fresh, after a GEMV
stack run, after gc, and after a 2 s idle (the idle alone leaves it ~8% slower). usage:
python scripts/dstep_gap.py plain|stack|stack_gc|stack_gconly|stack_sleep"""
import os, sys, time, gc
sys.path.insert(0, os.getcwd())
import torch
from paper_2410_08661_b200.qmodel import LLAMA2_7B
from paper_2410_08661_b200.model import QEFTDecoder
from paper_2410_08661_b200.generate import KVDecoder
from paper_2410_08661_b200.decode import LinearStack, llama_launch_groups, llama_stack_layers

def measure(tag):
    model = QEFTDecoder.synthetic(LLAMA2_7B, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
    for p in model.parameters(): p.requires_grad_(False)
    dec = KVDecoder(model, max_seq=545, capture=True)
    tok = torch.tensor([1])
    for p in range(512): dec.step(tok, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(32): dec.step(tok, 512 + i)
    e1.record(); torch.cuda.synchronize()
    print(tag, round(e0.elapsed_time(e1) / 32, 3), flush=True)
    del dec, model

mode = sys.argv[1]
if mode.startswith("stack"):
    layers = llama_stack_layers("7b", n_blocks=32)
    st = LinearStack(layers, n_cols=1, groups=llama_launch_groups(32))
    for _ in range(60): st.step()
    torch.cuda.synchronize()
    del st, layers
    torch.cuda.empty_cache()
    if mode in ("stack_gc", "stack_gconly"):
        gc.collect(); torch.cuda.empty_cache()
    if mode in ("stack_gc", "stack_sleep"):
        time.sleep(2)
measure(mode)
measure(mode + "_again")
