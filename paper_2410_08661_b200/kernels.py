"""Matrix-vector paths over the packed format (reference API, GPU compute).

Same names and contracts as pkg/src/qeft/kernels.py:38-186:
  matvec_structured / matvec_irregular / matvec_online_reorder /
  matvec_reference / matvec_dispatch, KernelStats, analytic_bytes,
  analytic_fmas, KernelPathOp.
Every path runs the B200 decode GEMV (libqeft_b200 `qeft_gemv`); the layout
variants differ only in the colmap gather the kernel applies while staging x.
Inputs/outputs are host numpy float32 like the reference; the device copy of
the layer comes from layer.device_layer (cached per record, ours or the
reference's own class, with the weak block re-synced from q.weak).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .errors import ShapeError
from .quantizer import LAYOUT_IRREGULAR, LAYOUT_STRUCTURED

PATH_STRUCTURED = "structured"
PATH_IRREGULAR = "irregular"
PATH_ONLINE = "online_reorder"
PATH_REFERENCE = "reference"


@dataclass
class KernelStats:
    elapsed_ns: int = 0
    bytes_read: int = 0
    fma: int = 0
    calls: int = 0
    path: str = ""

    def merge(self, other: "KernelStats") -> None:
        self.elapsed_ns += other.elapsed_ns
        self.bytes_read += other.bytes_read
        self.fma += other.fma
        self.calls += other.calls
        self.path = self.path or other.path


def analytic_bytes(q) -> int:
    """Reference accounting (kernels.py:54-58): packed + fp32 params + fp32 weak."""
    return len(q.packed) + 2 * 4 * q.oc * q.n_groups + 4 * q.oc * q.k


def analytic_fmas(q) -> int:
    return q.oc * q.m + 2 * q.oc * q.n_groups + q.oc * q.k


def b200_bytes(q, n_cols: int = 1) -> int:
    """Algorithmic HBM bytes of one B200 GEMV: codes + fp16 (scale, zero)
    + fp16 weak + fp16 x and y."""
    from .packing import row_bytes
    return (q.oc * row_bytes(q.m, q.bits) + 4 * q.oc * q.n_groups + 2 * q.oc * q.k
            + 2 * n_cols * (q.ic + q.oc))


def _bump(stats, q, t0, path, n=1):
    if stats is not None:
        stats.merge(KernelStats(elapsed_ns=time.perf_counter_ns() - t0,
                                bytes_read=n * analytic_bytes(q), fma=n * analytic_fmas(q),
                                calls=n, path=path))


def _run(q, xs: np.ndarray, perm=None) -> np.ndarray:
    """Columns of xs (ic, N) through the GEMV in chunks of 16; returns (oc, N) fp32."""
    import torch
    from .layer import device_layer
    dl = device_layer(q, "f16")
    if perm is not None:
        # matvec_online_reorder with an explicit permutation: a throwaway view
        # of the layer whose colmap composes the permutation (kernels.py:115-126)
        dl = _with_perm(q, dl, perm)
    # fp16 operands: scale x by an exact power of two so max|x| lands in [1, 2) (no overflow
    # past 65504, full fp16 precision for tiny inputs), divided back out of the fp32 result
    from .tuning import _pow2_scale
    sc = _pow2_scale(xs)
    xt = torch.from_numpy(np.ascontiguousarray(xs.T * np.float32(sc), np.float32)).cuda().to(torch.float16)
    out = torch.empty((xt.shape[0], q.oc), dtype=torch.float32, device="cuda")
    for s in range(0, xt.shape[0], 16):
        dl.gemv(xt[s:s + 16], out=out[s:s + 16])
    return (out.cpu().numpy().T / np.float32(sc)).astype(np.float32)


def _with_perm(q, dl, perm):
    import torch
    from .layer import DeviceLayer
    p = np.asarray(getattr(perm, "perm", perm), np.int64)
    if p.shape != (q.ic,):
        raise ShapeError("permutation does not match layer input width")
    colmap = np.full(dl.m_pad + dl.k_pad, -1, np.int32)
    colmap[:q.m] = p[:q.m]
    colmap[dl.m_pad:dl.m_pad + q.k] = p[q.m:]
    return DeviceLayer(oc=q.oc, ic=q.ic, k=q.k, bits=q.bits, g=q.g, qweight=dl.qweight, sz=dl.sz,
                       weak16=dl.weak16, colmap=torch.from_numpy(colmap).cuda(), dtype=dl.dtype,
                       sz16=dl.sz16)


def matvec_structured(q, x, stats: KernelStats | None = None) -> np.ndarray:
    if q.layout != LAYOUT_STRUCTURED:
        raise ShapeError("matvec_structured requires a structured layout")
    x = np.asarray(x, dtype=np.float32)
    if x.shape != (q.ic,):
        raise ShapeError(f"x shape {x.shape} != ({q.ic},)")
    if q.input_perm is not None:
        # structured path reads x in the layer's own (already reordered) order
        return matvec_online_reorder(q, x, np.arange(q.ic), stats)
    t0 = time.perf_counter_ns()
    y = _run(q, x[:, None])[:, 0]
    _bump(stats, q, t0, PATH_STRUCTURED)
    return y


def matvec_irregular(q, x, stats: KernelStats | None = None) -> np.ndarray:
    if q.layout != LAYOUT_IRREGULAR:
        raise ShapeError("matvec_irregular requires an irregular layout")
    x = np.asarray(x, dtype=np.float32)
    if x.shape != (q.ic,):
        raise ShapeError(f"x shape {x.shape} != ({q.ic},)")
    t0 = time.perf_counter_ns()
    y = _run(q, x[:, None])[:, 0]
    _bump(stats, q, t0, PATH_IRREGULAR)
    return y


def matvec_online_reorder(q, x_original, perm, stats: KernelStats | None = None) -> np.ndarray:
    x_original = np.asarray(x_original, dtype=np.float32)
    p = np.asarray(getattr(perm, "perm", perm), dtype=np.int64)
    if p.shape != (q.ic,):
        raise ShapeError("permutation does not match layer input width")
    t0 = time.perf_counter_ns()
    y = _run(q, x_original[:, None], perm=p)[:, 0]
    _bump(stats, q, t0, PATH_ONLINE)
    return y


def matvec_reference(q, x) -> np.ndarray:
    """Dense path: the device-dequantized matrix times x in fp64 on the GPU. The device
    dequant writes column colmap[j] = input_perm[qpos[j]], i.e. W in ORIGINAL input
    coordinates, so x is used as given (online layouts included)."""
    import torch
    from .layer import device_layer
    x = np.asarray(x, dtype=np.float64)
    w = device_layer(q, "f16").dequant_full().double()
    return (w @ torch.from_numpy(x).cuda()).cpu().numpy()


def native_path(q) -> str:
    if q.input_perm is not None:
        return PATH_ONLINE
    if q.layout == LAYOUT_STRUCTURED:
        return PATH_STRUCTURED
    return PATH_IRREGULAR


def matvec_dispatch(q, x, stats=None, path=None) -> np.ndarray:
    path = path or native_path(q)
    if path == PATH_REFERENCE:
        return matvec_reference(q, x).astype(np.float32)
    if path == PATH_ONLINE:
        return matvec_online_reorder(q, x, q.input_perm, stats)
    if path == PATH_STRUCTURED:
        return matvec_structured(q, x, stats)
    if path == PATH_IRREGULAR:
        return matvec_irregular(q, x, stats)
    raise ShapeError(f"unknown kernel path {path!r}")


class KernelPathOp:
    """Engine linear op (kernels.py:163-186): every activation column goes
    through the decode GEMV, 16 columns per launch."""

    def __init__(self, name, q, stats_map, reference=False):
        self.name = name
        self.q = q
        self.oc, self.ic = q.oc, q.ic
        self.reference = reference
        self.stats = stats_map.setdefault(name, KernelStats())

    def apply(self, x2d):
        x2d = np.asarray(x2d, np.float32)
        if self.reference:
            return np.stack([matvec_reference(self.q, x2d[:, j]).astype(np.float32)
                             for j in range(x2d.shape[1])], axis=1) if x2d.shape[1] else \
                np.zeros((self.oc, 0), np.float32)
        t0 = time.perf_counter_ns()
        if self.q.input_perm is not None:
            y = _run(self.q, x2d, perm=self.q.input_perm)
        else:
            y = _run(self.q, x2d)
        _bump(self.stats, self.q, t0, native_path(self.q), n=x2d.shape[1])
        return y

    def forward_train(self, x2d):
        return self.apply(x2d), None

    def backward(self, state, dy2d, need_weight_grad=True):
        raise ShapeError("kernel-path ops are inference-only")
