"""GEMV microbenchmark: per-launch time of each 7B shape, graph of 32 distinct
layers (weights stream from HBM), n = 1 and 16."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import LinearStack, random_layer

peak = 6553.0
res = []
for n in (1, 4, 16):
    for (oc, ic) in ((4096, 4096), (11008, 4096), (4096, 11008), (5120, 5120), (8192, 28672)):
        nl = 32 if oc * ic < 1e8 else 8
        layers = [random_layer(oc, ic, 128, 4, 128, "f16", seed=b) for b in range(nl)]
        st = LinearStack(layers, n_cols=n)
        for _ in range(3):
            st.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        reps = 10
        for _ in range(reps):
            st.step()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / (reps * nl)
        b = st.bytes_per_step() / nl
        res.append(dict(n=n, shape=[oc, ic], us=t * 1e6, gbs=b / t / 1e9, frac=b / t / 1e9 / peak))
        print(json.dumps(res[-1]), flush=True)
        del st, layers
        torch.cuda.empty_cache()
