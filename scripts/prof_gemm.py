"""One QEFTLinear fwd + bwd at T tokens (for ncu capture of gemm fwd/dgrad/wgrad)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer
from paper_2410_08661_b200.qlinear import QEFTLinear
oc, ic = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x4096").split("x"))
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
lin = QEFTLinear(random_layer(oc, ic, 128, 4, 128, "f16", seed=1))
x = torch.randn(T, ic, device="cuda", dtype=torch.float16, requires_grad=True)
dy = torch.randn(T, oc, device="cuda", dtype=torch.float16)
for _ in range(2):
    lin(x).backward(dy)
torch.cuda.synchronize()
