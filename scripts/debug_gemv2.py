"""Isolate GEMV cases: each case runs in its own subprocess with a timeout and prints the
max error against an fp64 product over the device-dequantized weights.
usage: python scripts/debug_gemv2.py            (driver)
       python scripts/debug_gemv2.py one OC IC K BITS G N S   (single case)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(oc, ic, k, bits, g, n, S, dtype="f16"):
    import numpy as np
    import torch
    from paper_2410_08661_b200 import quantizer
    from paper_2410_08661_b200.layer import device_layer
    if S:
        os.environ["QEFT_GEMV2_S"] = str(S)
    rng = np.random.default_rng(oc + ic + k)
    w = (rng.standard_normal((oc, ic)) * 0.02).astype(np.float32)
    q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn")
    dl = device_layer(q, dtype)
    W = dl.dequant_full().double()
    x = torch.randn(n, ic, device="cuda").to(dl.tdtype)
    y = dl.gemv(x, out_f32=True)
    torch.cuda.synchronize()
    ref = x.double() @ W.T
    err = float((y.double() - ref).abs().max() / max(1.0, float(ref.abs().max())))
    y2 = dl.gemv(x, out_f32=True)
    same = bool(torch.equal(y, y2))
    bad = ((y.double() - ref).abs() > 1e-2 * max(1.0, float(ref.abs().max()))).nonzero()
    print(f"case oc={oc} ic={ic} k={k} bits={bits} g={g} n={n} S={S}: err {err:.3e} det {same} "
          f"bad {bad.shape[0]} first {bad[:6].tolist()}")


CASES = [
    (4096, 4096, 128, 4, 128, 1, 1), (4096, 4096, 128, 4, 128, 1, 2), (4096, 4096, 128, 4, 128, 1, 4),
    (4096, 4096, 128, 3, 128, 1, 1), (4096, 4096, 128, 3, 128, 1, 4),
    (4096, 4096, 16, 4, 64, 1, 0), (4096, 4096, 16, 4, 64, 1, 1),
    (48, 8192, 16, 4, 128, 1, 0), (48, 8192, 16, 4, 128, 1, 1),
    (4096, 4096, 8, 4, 32, 1, 0),
    (512, 1024, 128, 4, 128, 1, 1), (512, 1024, 128, 4, 128, 4, 1), (512, 1024, 128, 4, 128, 16, 1),
    (512, 1024, 128, 4, 128, 1, 2), (4096, 11008, 128, 4, 128, 1, 0),
]

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one(*[int(v) for v in sys.argv[2:9]])
        sys.exit(0)
    for c in CASES:
        try:
            r = subprocess.run([sys.executable, __file__, "one", *map(str, c)], capture_output=True, text=True,
                               timeout=90)
            out = (r.stdout.strip().splitlines() or [""])[-1]
            print(out if r.returncode == 0 else f"case {c}: rc {r.returncode} {r.stderr[-600:]}", flush=True)
        except subprocess.TimeoutExpired:
            print(f"case {c}: TIMEOUT", flush=True)
