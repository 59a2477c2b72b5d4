"""One decode launch of the given type (qkv | o | gate_up | down) of a 7B block, a few times
(for ncu capture of the kernel the bench times). usage: prof_decode.py TYPE [N_COLS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import LAUNCHES
from paper_2410_08661_b200.decode import LinearStack, random_layer
name = sys.argv[1]
n_cols = int(sys.argv[2]) if len(sys.argv) > 2 else 1
shapes = dict((n, s) for n, s, _ in LAUNCHES)[name]
layers = [random_layer(oc, ic, 128, 4, 128, "f16", seed=i) for i, (oc, ic) in enumerate(shapes)]
st = LinearStack(layers, n_cols=n_cols, use_graph=False, groups=[list(range(len(layers)))])
for _ in range(4):
    st.step()
torch.cuda.synchronize()
