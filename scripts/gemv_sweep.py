"""GEMV tuning sweep: per-launch time of each shape under a CUDA graph of
distinct layers (weights stream from HBM), for RBW / smem-budget settings."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08661_b200.decode import LinearStack, random_layer

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6460.0
shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 28672), (28672, 8192)]
ns = [int(v) for v in os.environ.get("NS", "1,16").split(",")]
rbws = os.environ.get("RBWS", "0,1,2").split(",")
smems = os.environ.get("SMEMS", "0").split(",")
for n in ns:
    for (oc, ic) in shapes:
        nl = 32 if oc * ic < 1e8 else 6
        layers = [random_layer(oc, ic, 128, 4, 128, "f16", seed=b) for b in range(nl)]
        for rbw, sm in itertools.product(rbws, smems):
            for k, v in (("QEFT_GEMV_RBW", rbw), ("QEFT_GEMV_SMEM", sm)):
                if v == "0":
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            st = LinearStack(layers, n_cols=n)
            for _ in range(3):
                st.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 10
            e0.record()
            for _ in range(reps):
                st.step()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / (reps * nl)
            b = st.bytes_per_step() / nl
            print(json.dumps(dict(n=n, shape=[oc, ic], rbw=rbw, smem=sm, us=round(t * 1e6, 2),
                                  gbs=round(b / t / 1e9, 1), frac=round(b / t / 1e9 / peak, 3))), flush=True)
            del st
        del layers
        torch.cuda.empty_cache()
