"""Isolated wgrad timing (CUDA events, no PDL neighbours): dW_weak for the 7B shapes at T=2048,
for the library at QEFT_LIB_PATH; QEFT_WGRAD_SPLITS overrides the split count."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
T = 2048
res = {}
for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
    dl = random_layer(oc, ic, 128, 4, 128, "bf16", seed=5)
    x = torch.randn(T, ic, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(T, oc, device="cuda", dtype=torch.bfloat16)
    xw = dl.gather_weak(x)
    out = torch.zeros(oc, 128, device="cuda")
    fn = lambda: dl.gemm_wgrad_weak(dy, xw, out=out, accumulate=True)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    # CUDA graph of 50 calls: device time without the per-call host overhead
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(50): fn()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    res[f"wgrad {oc}"] = round(us, 1)
    res[f"GB/s {oc}"] = round(T * oc * 2 / us / 1e3)
print(os.environ.get("QEFT_LIB_PATH", "default"), os.environ.get("QEFT_WGRAD_SPLITS", ""), json.dumps(res))
