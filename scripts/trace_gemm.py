"""Per-CTA globaltimer trace of one fwd GEMM launch (qeft_gemv_trace slots are shared with the
GEMM): prologue, first MMA, mainloop, epilogue, per CTA. usage: trace_gemm.py [OC IC T] [f16]"""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_08661_b200 import _lib
from paper_2410_08661_b200.decode import random_layer
oc, ic, T = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 2048)))
mode = sys.argv[4] if len(sys.argv) > 4 else "fwd"
dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=5)
x = torch.randn(T, ic if mode == "fwd" else oc, device="cuda", dtype=torch.float16)
fn = (lambda: dl.gemm_fwd(x)) if mode == "fwd" else (lambda: dl.gemm_dgrad(x))
for _ in range(3):
    fn()
torch.cuda.synchronize()
L = _lib.lib()
L.qeft_gemv_trace(2, None)
fn(); fn()
torch.cuda.synchronize()
buf = np.zeros(2 * 512 * 8, np.uint64)
L.qeft_gemv_trace(0, buf.ctypes.data_as(ctypes.c_void_p))
tr = buf.reshape(2, 512, 8).astype(np.int64)[1]
v = tr[tr[:, 0] > 0]
t0 = v[:, 0].min()
rel = (v - t0) / 1e3  # us
names = ["start", "setup", "mma0", "mma_last", "tfull0", "epi_end", "prod0", "end"]
out = {"shape": [oc, ic, T], "mode": mode, "ctas": int(len(v)), "kernel_us": float(rel[:, 7].max())}
for i, n in enumerate(names):
    col = rel[:, i]
    out[n] = [round(float(np.min(col)), 2), round(float(np.median(col)), 2), round(float(np.max(col)), 2)]
mm = rel[v[:, 2] > 0]  # CTAs that issued MMAs (a pair's leader only)
out["mainloop_us"] = [round(float(x), 2) for x in np.percentile(mm[:, 3] - mm[:, 2], [0, 50, 100])]
out["epilogue_us"] = [round(float(x), 2) for x in np.percentile(mm[:, 5] - mm[:, 3], [0, 50, 100])]
for i in (2, 3):
    out[names[i]] = [round(float(np.min(mm[:, i])), 2), round(float(np.median(mm[:, i])), 2), round(float(np.max(mm[:, i])), 2)]
print(json.dumps(out))
