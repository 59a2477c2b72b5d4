"""Decode-step GEMV stack: a model's quantized linears run as one CUDA graph.

Public API for batch 1..16 decoding over many QEFT layers (the analog of the
reference's per-token loop in `bench_generate`, pkg/src/qeft/kernels.py:
197-228, restricted to the linear layers this package owns):

    stack = LinearStack(layers, n_cols=1)
    y_host = stack.run(x_host)          # H2D x, graph replay, D2H outputs

`LinearStack.step()` replays the captured graph on device-resident inputs.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ShapeError
from .layer import GEMV_WORKSPACE, DeviceLayer, _pad, make_sz16, torch_dtype

LLAMA_SHAPES = {
    # name -> (oc, ic) for one decoder block
    "7b": [("wq", 4096, 4096), ("wk", 4096, 4096), ("wv", 4096, 4096), ("wo", 4096, 4096),
           ("w_up", 11008, 4096), ("w_gate", 11008, 4096), ("w_down", 4096, 11008)],
    "13b": [("wq", 5120, 5120), ("wk", 5120, 5120), ("wv", 5120, 5120), ("wo", 5120, 5120),
            ("w_up", 13824, 5120), ("w_gate", 13824, 5120), ("w_down", 5120, 13824)],
    "70b": [("wq", 8192, 8192), ("wk", 1024, 8192), ("wv", 1024, 8192), ("wo", 8192, 8192),
            ("w_up", 28672, 8192), ("w_gate", 28672, 8192), ("w_down", 8192, 28672)],
}
N_BLOCKS = {"7b": 32, "13b": 40, "70b": 80}


def random_layer(oc, ic, k=128, bits=4, g=128, dtype="f16", seed=0, device="cuda"):
    """A synthetic layer directly in the B200 layout: codes
    uniform in [0, 2^b), scale 1e-3 + 0.01|N(0,1)|, zero N(0, 0.05), weak N(0, 0.02).
    GEMV time does not depend on the values."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    m = ic - k
    m_pad, k_pad, oc_pad = _pad(m, 128), _pad(k, 64), _pad(oc, 16)
    ng = max(1, -(-m // g))
    nbytes = int(_lib.lib().qeft_qweight_bytes(oc, m, bits))
    qweight = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=device, generator=gen)
    td = torch_dtype(dtype)
    s = 1e-3 + 0.01 * torch.randn(oc_pad, ng, device=device, generator=gen).abs()
    z = 0.05 * torch.randn(oc_pad, ng, device=device, generator=gen)
    sz = torch.stack([s, z], -1).reshape(oc_pad // 16, 16, ng, 2).permute(0, 2, 1, 3).contiguous()
    # weak16 in row-block tiles [oc_pad/16][k_pad/64][16][64] (csrc/qeft_common.cuh weak_off)
    weak16 = (0.02 * torch.randn(oc_pad // 16, k_pad // 64, 16, 64, device=device, generator=gen)).to(td)
    if k_pad:
        col = (torch.arange(k_pad // 64, device=device)[:, None] * 64 + torch.arange(64, device=device))
        weak16.masked_fill_((col >= k)[None, :, None, :], 0)
    weak16 = weak16.reshape(oc_pad, k_pad)
    colmap = torch.full((m_pad + k_pad,), -1, dtype=torch.int32, device=device)
    colmap[:m] = torch.arange(m, dtype=torch.int32, device=device)
    colmap[m_pad:m_pad + k] = torch.arange(m, ic, dtype=torch.int32, device=device)
    return DeviceLayer(oc=oc, ic=ic, k=k, bits=bits, g=g, qweight=qweight, sz=sz.reshape(-1),
                       weak16=weak16, colmap=colmap, dtype=dtype,
                       structured_fast=(m % 8 == 0 and ic % 8 == 0),
                       sz16=make_sz16(s[:oc].float(), z[:oc].float(), oc, m, g))


def gemv_multi(layers, x, outs, norm_gain=None):
    """One decode-GEMV launch over layers that read the same x (qeft_gemv_multi): a
    decoder's q/k/v or gate/up. outs[l] is layer l's (n, oc_l) output. norm_gain (fp32 [ic]):
    x is RMS-normalised inside the launch first (qeft_gemv_multi_rmsnorm), bit-identical to
    fused.rms_norm followed by this call."""
    n = x.shape[0]
    L = _lib.lib()
    arr = (ctypes.POINTER(_lib.QeftLinearT) * len(layers))(*[l.cptr for l in layers])
    ys = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    ldy = outs[0].stride(0) if n > 1 else max(l.oc for l in layers)
    if any((o.stride(0) if n > 1 else ldy) != ldy for o in outs):
        raise ShapeError("gemv_multi: outputs need a common row stride")
    wsb = sum(int(L.qeft_gemv_workspace_bytes(l.cptr, n)) for l in layers)
    ws = GEMV_WORKSPACE.get(wsb, x.device)
    ldx = x.stride(0) if n > 1 else layers[0].ic
    yf = 1 if outs[0].dtype.itemsize == 4 else 0
    if norm_gain is not None:
        g = norm_gain.contiguous().float()
        _lib.check(L.qeft_gemv_multi_rmsnorm(ctypes.cast(arr, ctypes.c_void_p), len(layers), _lib.ptr(x), ldx,
                                             _lib.ptr(g), ctypes.cast(ys, ctypes.c_void_p), ldy, yf, n,
                                             _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gemv_multi_rmsnorm")
        return outs
    _lib.check(L.qeft_gemv_multi(ctypes.cast(arr, ctypes.c_void_p), len(layers), _lib.ptr(x), ldx,
                                 ctypes.cast(ys, ctypes.c_void_p), ldy, yf, n, _lib.ptr(ws), ws.numel(),
                                 _lib.stream_ptr()), "gemv_multi")
    return outs


def llama_launch_groups(n_blocks):
    """Layers of one decode launch per block of llama_stack_layers' order (wq, wk, wv, wo,
    w_up, w_gate, w_down): q/k/v share x, so do gate/up."""
    groups = []
    for b in range(n_blocks):
        i = 7 * b
        groups += [[i, i + 1, i + 2], [i + 3], [i + 4, i + 5], [i + 6]]
    return groups


def llama_stack_layers(model="7b", k=128, bits=4, g=128, dtype="f16", n_blocks=None, seed=0):
    layers = []
    for b in range(n_blocks if n_blocks is not None else N_BLOCKS[model]):
        for i, (_, oc, ic) in enumerate(LLAMA_SHAPES[model]):
            layers.append(random_layer(oc, ic, k, bits, g, dtype, seed=seed * 100003 + b * 7 + i))
    return layers


class LinearStack:
    """Run every layer's GEMV once per step (decode of one token batch)."""

    def __init__(self, layers, n_cols=1, use_graph=True, groups=None):
        import torch
        self.layers = layers
        self.n = n_cols
        # launch groups: layers sharing x in one qeft_gemv_multi launch (default: one per layer)
        self.groups = groups if groups is not None else [[i] for i in range(len(layers))]
        dev = layers[0].device
        td = layers[0].tdtype
        self.ics = sorted({l.ic for l in layers})
        # one input buffer per distinct input width, one output per layer
        self.x = {ic: torch.zeros((n_cols, ic), dtype=td, device=dev) for ic in self.ics}
        # every layer's output is a column slice of ONE (n, sum oc) buffer: one D2H per step
        tot = sum(l.oc for l in layers)
        self.y_all = torch.empty((n_cols, tot), dtype=td, device=dev)
        offs = np.concatenate([[0], np.cumsum([l.oc for l in layers])]).astype(int)
        self.y = [self.y_all[:, offs[i]:offs[i + 1]] for i in range(len(layers))]
        self.y_flat_host = torch.empty(tot * n_cols, dtype=td).pin_memory()
        self.x_host = {ic: torch.empty((n_cols, ic), dtype=td).pin_memory() for ic in self.ics}
        self.graph = None
        # warm the workspace and the kernels once eagerly
        self._launch()
        torch.cuda.synchronize()
        if use_graph:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._launch()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self._launch()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            self.graph = g

    def _launch(self):
        for grp in self.groups:
            if len(grp) == 1:
                l = self.layers[grp[0]]
                l.gemv(self.x[l.ic], out=self.y[grp[0]])
            else:
                gemv_multi([self.layers[i] for i in grp], self.x[self.layers[grp[0]].ic],
                           [self.y[i] for i in grp])

    def step(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()

    def launches_per_step(self) -> int:
        return len(self.groups)

    def bytes_per_step(self) -> int:
        """Algorithmic HBM bytes (weights + fp16 x and y)."""
        return sum(l.weight_bytes() + 2 * self.n * (l.ic + l.oc) for l in self.layers)

    def run(self, x_host: dict | np.ndarray | None = None):
        """End-to-end step through host memory: copy inputs in, replay, copy all
        outputs back (pinned buffers). Returns the host output buffer."""
        import torch
        if x_host is not None:
            for ic in self.ics:
                src = x_host[ic] if isinstance(x_host, dict) else x_host
                self.x_host[ic].copy_(torch.as_tensor(src)[..., :ic] if not isinstance(x_host, dict) else torch.as_tensor(src))
        for ic in self.ics:
            self.x[ic].copy_(self.x_host[ic], non_blocking=True)
        self.step()
        self.y_flat_host.copy_(self.y_all.reshape(-1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.y_flat_host

    def h2d_bytes(self) -> int:
        return sum(2 * self.n * ic for ic in self.ics)

    def d2h_bytes(self) -> int:
        return sum(2 * self.n * l.oc for l in self.layers)
