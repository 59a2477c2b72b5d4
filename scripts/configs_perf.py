"""Performance of the BASELINE.json parity configs (device time, CUDA events):
  configs[3]: LLaMA-2-13B-shaped 3-bit prefill GEMM (fwd, dX) at T = 512, 2048;
  configs[4]: LLaMA-2-70B-shaped 4-bit layers, weak-column sweep k = 16..256: decode GEMV GB/s (N=1).
Writes one JSON object (stdout)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import LinearStack, random_layer


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


out = {"gemm_13b_3bit": [], "gemv_70b_k_sweep": []}
for oc, ic in ((5120, 5120), (13824, 5120), (5120, 13824)):
    dl = random_layer(oc, ic, 128, 3, 128, "bf16", seed=1)
    for T in (512, 2048):
        x = torch.randn(T, ic, device="cuda", dtype=torch.bfloat16)
        dy = torch.randn(T, oc, device="cuda", dtype=torch.bfloat16)
        f = 2.0 * T * oc * ic
        out["gemm_13b_3bit"].append({"shape": [oc, ic], "T": T,
                                     "fwd_tflops": f / timed(lambda: dl.gemm_fwd(x)) / 1e12,
                                     "dgrad_tflops": f / timed(lambda: dl.gemm_dgrad(dy)) / 1e12})
        del x, dy
    del dl
for oc, ic in ((28672, 8192), (8192, 28672)):
    for k in (16, 32, 64, 128, 256):
        # 8 distinct layers in one graph so the weights stream from HBM (8 x ~120 MB >> L2)
        layers = [random_layer(oc, ic, k, 4, 128, "f16", seed=s) for s in range(8)]
        st = LinearStack(layers, n_cols=1)
        sec = timed(st.step, reps=20)
        out["gemv_70b_k_sweep"].append({"shape": [oc, ic], "k": k, "gbs": st.bytes_per_step() / sec / 1e9,
                                        "us_per_layer": sec / len(layers) * 1e6})
        del st, layers
        torch.cuda.empty_cache()
print(json.dumps(out))
