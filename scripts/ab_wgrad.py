"""wgrad timing for the 7B shapes at T=2048 (CUDA events), for QEFT_WGRAD_SPLITS tuning."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
T = 2048
res = {}
for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
    dl = random_layer(oc, ic, 128, 4, 128, "bf16", seed=5)
    xw = torch.randn(T, 128, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(T, oc, device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(oc, 128, device="cuda")
    fn = lambda: dl.gemm_wgrad_weak(dy, xw, out=out, accumulate=True)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    res[f"{oc}x{ic}"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
print(os.environ.get("QEFT_WGRAD_SPLITS", "auto"), "us:", json.dumps(res))
