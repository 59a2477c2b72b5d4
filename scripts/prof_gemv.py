"""A few eager GEMV launches per shape, for ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import random_layer

shapes = [(int(a), int(b)) for a, b in (s.split("x") for s in sys.argv[1].split(","))] if len(sys.argv) > 1 else [(4096, 4096)]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for oc, ic in shapes:
    ls = [random_layer(oc, ic, 128, 4, 128, "f16", seed=i) for i in range(4)]
    x = torch.randn(n, ic, device="cuda").half()
    for l in ls:
        l.gemv(x)
    torch.cuda.synchronize()
