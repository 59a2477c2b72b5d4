"""GPU debug: GEMV vs device dequant reference over a grid of shapes; prints
max error and where it occurs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_08661_b200 import quantizer

cases = [
    (1000, 2176, 128, 4, 128, "f16", 1), (1000, 2176, 128, 4, 128, "f16", 16),
    (1024, 2176, 128, 4, 128, "f16", 1), (1000, 2176, 128, 4, 128, "f16", 5),
    (200, 1100, 12, 4, 128, "bf16", 3), (200, 1100, 12, 3, 128, "bf16", 3),
    (200, 1100, 12, 4, 40, "f16", 3), (200, 1100, 12, 3, 24, "bf16", 3),
    (256, 1024, 0, 4, 128, "f16", 1), (64, 1152, 128, 4, 128, "f16", 1),
    (16, 40, 4, 4, 8, "f16", 1), (6, 12, 3, 4, 4, "f16", 1), (30, 70, 5, 3, 7, "f16", 1),
    (64, 256, 64, 4, 64, "f16", 1), (64, 256, 64, 4, 64, "bf16", 1),
]
for (oc, ic, k, bits, g, dt, n) in cases:
    rng = np.random.default_rng(oc + ic)
    w = (rng.standard_normal((oc, ic)) * 0.05).astype(np.float32)
    q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn")
    dl = q.device(dt)
    x = torch.randn(n, ic, device="cuda").to(dl.tdtype)
    y = dl.gemv(x, out_f32=True)
    dq = dl.dequant_full().double()
    host = torch.from_numpy(q.dequant_full()).cuda().double()
    ref = x.double() @ dq.T
    err = (y.double() - ref).abs()
    rel = float(err.max() / max(1.0, float(ref.abs().max())))
    dqerr = float((dq - host).abs().max())
    i = int(err.argmax())
    print(f"oc={oc} ic={ic} k={k} bits={bits} g={g} {dt} n={n}: rel={rel:.3e} dq_vs_host={dqerr:.2e} "
          f"worst at (n={i // oc}, row={i % oc}) y={float(y.view(-1)[i]):.4f} ref={float(ref.view(-1)[i]):.4f} nan={bool(torch.isnan(y).any())}")
