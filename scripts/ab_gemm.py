"""A/B timing of the fwd/dgrad GEMMs (CUDA events) for the library at QEFT_LIB_PATH."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
DT = os.environ.get("AB_DT", "f16")
TD = torch.float16 if DT == "f16" else torch.bfloat16
res = {}
SHAPES = [(4096, 4096, 2048), (11008, 4096, 2048), (4096, 11008, 2048), (5120, 5120, 512), (13824, 5120, 512),
          (5120, 13824, 512)]
for oc, ic, T in SHAPES:
    dl = random_layer(oc, ic, 128, 4, 128, DT, seed=5)
    x = torch.randn(T, ic, device="cuda", dtype=TD)
    dy = torch.randn(T, oc, device="cuda", dtype=TD)
    for name, fn in (("fwd", lambda: dl.gemm_fwd(x)), ("dgrad", lambda: dl.gemm_dgrad(dy))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 20 / 1e3
        res[f"{name} {oc}x{ic} T{T}"] = round(2 * T * oc * ic / s / 1e12)
print("SK=" + os.environ.get("QEFT_GEMM_SK", "auto"), json.dumps(res))
