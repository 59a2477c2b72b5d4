"""One 7B-shaped fwd GEMM (4096 x 4096, T = 2048, f16) per call, for ncu A/B of the tile schedule."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
oc, ic, T = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 2048)))
dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=5)
x = torch.randn(T, ic, device="cuda", dtype=torch.float16)
for _ in range(4):
    dl.gemm_fwd(x)
torch.cuda.synchronize()
