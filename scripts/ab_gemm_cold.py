"""fwd/dgrad GEMM TFLOP/s with L2 flushed before every launch (the step's situation: each
layer's weights and activations come from HBM). usage: ab_gemm_cold.py [package_root]"""
import os, sys, json
root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.abspath(root))
import torch
from paper_2410_08661_b200.decode import random_layer
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
res = {}
for oc, ic, T in ((4096, 4096, 2048), (11008, 4096, 2048), (4096, 11008, 2048)):
    dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=5)
    x = torch.randn(T, ic, device="cuda", dtype=torch.float16)
    dy = torch.randn(T, oc, device="cuda", dtype=torch.float16)
    for name, fn in (("fwd", lambda: dl.gemm_fwd(x)), ("dgrad", lambda: dl.gemm_dgrad(dy))):
        for _ in range(3): fn()
        tot = 0.0
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) / 1e3
        res[f"{name} {oc}x{ic}"] = round(2 * T * oc * ic / (tot / 10) / 1e12)
print(root, json.dumps(res))
