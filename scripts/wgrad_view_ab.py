"""wgrad from the strided weak-column view of x vs from a gathered copy (7B shapes, f16)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
def timed(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
    dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=5)
    T = 2048
    x = torch.randn(T, ic, device="cuda", dtype=torch.float16)
    dy = torch.randn(T, oc, device="cuda", dtype=torch.float16)
    w = torch.zeros(oc, dl.k, device="cuda")
    view = x[:, dl.m:dl.m + dl.k]
    gath = dl.gather_weak(x)
    r = {"shape": [oc, ic], "view_us": round(timed(lambda: dl.gemm_wgrad_weak(dy, view, out=w, accumulate=True)), 1),
         "gathered_us": round(timed(lambda: dl.gemm_wgrad_weak(dy, gath, out=w, accumulate=True)), 1),
         "gather_us": round(timed(lambda: dl.gather_weak(x)), 1)}
    print(json.dumps(r), flush=True)
