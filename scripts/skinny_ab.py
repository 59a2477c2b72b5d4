"""Batched decode shapes (n = 4..16 columns): the bulk-copy GEMV against the tcgen05 GEMM
(whole tiles / stream-K) on the 7B layers, CUDA events, L2 flushed before each launch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200 import _lib
from paper_2410_08661_b200.decode import random_layer
L = _lib.lib()
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
def timed(fn):
    for _ in range(3): fn()
    tot = 0.0
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / 10 * 1e3  # us
out = []
for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
    dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=3)
    wb = dl.weight_bytes() if hasattr(dl, "weight_bytes") else None
    for n in (4, 8, 16, 32, 64):
        x = torch.randn(n, ic, device="cuda", dtype=torch.float16)
        r = {"shape": [oc, ic], "n": n, "gemv_us": round(timed(lambda: dl.gemv(x)), 2) if n <= 16 else None}
        for sk in (0, 1):
            L.qeft_gemm_set_schedule(0, sk)
            r[f"gemm_sk{sk}_us"] = round(timed(lambda: dl.gemm_fwd(x)), 2)
        L.qeft_gemm_set_schedule(0, -1)
        out.append(r)
        print(json.dumps(r), flush=True)
