"""Per-CTA globaltimer trace of consecutive decode GEMV launches (qeft_gemv_trace)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_08661_b200 import _lib
from paper_2410_08661_b200.decode import LinearStack, llama_launch_groups, llama_stack_layers

use_graph = "--graph" in sys.argv
layers = llama_stack_layers("7b", n_blocks=2)
L = _lib.lib()
SL = 8
if use_graph:
    # the trace pointers are baked into the captured launches: arm eager + warm + captured slots
    L.qeft_gemv_trace(3 * SL, None)
    st = LinearStack(layers, n_cols=1, use_graph=True, groups=llama_launch_groups(2))
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    buf = np.zeros(3 * SL * 512 * 8, np.uint64)
    L.qeft_gemv_trace(0, buf.ctypes.data_as(ctypes.c_void_p))
    tr = buf.reshape(3 * SL, 512, 8).astype(np.int64)[2 * SL:]
else:
    st = LinearStack(layers, n_cols=1, use_graph=False, groups=llama_launch_groups(2))
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    L.qeft_gemv_trace(SL, None)
    st.step()
    torch.cuda.synchronize()
    buf = np.zeros(SL * 512 * 8, np.uint64)
    L.qeft_gemv_trace(0, buf.ctypes.data_as(ctypes.c_void_p))
    tr = buf.reshape(SL, 512, 8).astype(np.int64)
names = ["qkv", "o", "gate_up", "down"] * 2
t00 = tr[0][tr[0][:, 0] > 0][:, 0].min()
prev_end = None
for s in range(SL):
    v = tr[s][tr[s][:, 0] > 0] - t00
    if not len(v):
        continue
    start, end = v[:, 0].min(), v[:, 6].max()
    med = lambda a: float(np.median(a))
    print(f"{names[s]:8s} ctas {len(v):3d} start {start/1e3:7.2f} end {end/1e3:7.2f} dur {(end-start)/1e3:6.2f} us | "
          f"start-spread {(v[:,0].max()-start)/1e3:5.2f} issue {med(v[:,7]-v[:,0])/1e3:5.2f} wait {med(v[:,1]-v[:,7])/1e3:5.2f} stage {med(v[:,2]-v[:,1])/1e3:5.2f} "
          f"first-data {med(v[:,3]-v[:,0])/1e3:5.2f} loop {med(v[:,4]-v[:,2])/1e3:5.2f} (max {(v[:,4]-v[:,2]).max()/1e3:5.2f}) "
          f"x-landed {med(v[:,5]-v[:,1])/1e3:5.2f} epi {med(v[:,6]-v[:,4])/1e3:5.2f} | gap {((start-prev_end)/1e3 if prev_end is not None else 0):5.2f}")
    prev_end = end
