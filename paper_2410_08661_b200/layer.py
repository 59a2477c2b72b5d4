"""Device-resident QEFT layer in the B200 tile layout, and the torch-level
calls into the CUDA library (GEMV / GEMM / dequant).

HBM layout of one layer (all on one GPU; see csrc/qeft_common.cuh):
  qweight  uint8   (oc_pad/16) row-blocks x K-tiles of 512 B (4-bit) / 768 B (3-bit)
  sz       fp32    (scale, zero) pairs [oc_pad/16][ng][16][2] (the reference's storage precision;
                   read by the GEMMs, the dequant and the generic-g GEMV)
  sz16     fp16    decode-GEMV copy of (scale, zero): half2 [oc_pad/16][ng16][8][2], 4 B per row
                   and group, ng16 = ceil(m_pad/g)
  weak16   dtype   [oc_pad][k_pad]  (the trainable block's kernel shadow)
  colmap   int32   [m_pad + k_pad]  B200 K position -> input column (-1 padding)
  weak32   fp32    [oc][k]          trainable master (a view into the DP bucket
                                     when the layer belongs to a model)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ShapeError

_DT = {"f16": _lib.QEFT_F16, "bf16": _lib.QEFT_BF16}


def _pad(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def torch_dtype(dtype: str):
    import torch
    return {"f16": torch.float16, "bf16": torch.bfloat16}[dtype]


class _Workspace:
    """Zero-initialised scratch shared by consecutive calls on one device.
    Kernels that use split-K counters leave them zeroed again."""

    def __init__(self):
        self.buf = {}

    def get(self, nbytes: int, device):
        import torch
        key = (str(device), torch.cuda.current_stream(device).cuda_stream)
        b = self.buf.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self.buf[key] = b
        return b


WORKSPACE = _Workspace()
# the decode GEMV's scratch: its head holds split-K row-block counters that must stay zero
# between calls, so it is never shared with the GEMMs' gather buffers
GEMV_WORKSPACE = _Workspace()


def make_sz16(scales, zeros, oc: int, m: int, g: int):
    """fp32 scales/zeros CUDA tensors [oc][ng] -> the GEMV's fp16 (scale, zero) copy."""
    import torch
    L = _lib.lib()
    out = torch.zeros(max(int(L.qeft_sz16_bytes(oc, m, g)), 16), dtype=torch.uint8, device=scales.device)
    if m > 0:
        _lib.check(L.qeft_pack_sz16(_lib.ptr(scales.contiguous()), _lib.ptr(zeros.contiguous()), oc, m, g,
                                    _lib.ptr(out), _lib.stream_ptr()), "pack_sz16")
    return out


class DeviceLayer:
    """A QuantizedLinear converted to the B200 layout on the current GPU."""

    def __init__(self, *, oc, ic, k, bits, g, qweight, sz, weak16, colmap, dtype="f16",
                 weak32=None, structured_fast=False, source_id=None, sz16=None):
        import torch
        self.oc, self.ic, self.k, self.bits, self.g = oc, ic, k, bits, g
        self.m = ic - k
        self.ng = max(1, -(-self.m // g)) if self.m > 0 else 0
        self.m_pad, self.k_pad, self.oc_pad = _pad(self.m, 128), _pad(k, 64), _pad(oc, 16)
        self.dtype = dtype
        self.tdtype = torch_dtype(dtype)
        self.qweight, self.sz, self.weak16, self.colmap = qweight, sz, weak16, colmap
        self.sz16 = sz16
        self.weak32 = weak32
        self.structured_fast = structured_fast
        self.source_id = source_id
        self._refresh_struct()

    def _refresh_struct(self):
        s = _lib.QeftLinearT()
        s.oc, s.ic, s.k, s.bits, s.g = self.oc, self.ic, self.k, self.bits, self.g
        s.m, s.ng, s.m_pad, s.k_pad, s.oc_pad = self.m, self.ng, self.m_pad, self.k_pad, self.oc_pad
        s.act_dtype = _DT[self.dtype]
        s.flags = _lib.QEFT_FLAG_STRUCTURED_FAST if self.structured_fast else 0
        s.qweight = self.qweight.data_ptr()
        s.sz = self.sz.data_ptr()
        s.weak16 = self.weak16.data_ptr() if self.weak16 is not None and self.weak16.numel() else None
        s.colmap = self.colmap.data_ptr()
        s.sz16 = self.sz16.data_ptr() if self.sz16 is not None else None
        self.cstruct = s
        self.cptr = ctypes.pointer(s)

    @property
    def device(self):
        return self.qweight.device

    # ------------------------------------------------------------------
    @classmethod
    def from_quantized(cls, q, dtype="f16", device="cuda"):
        """Upload + repack a QuantizedLinear (ours or the reference's record) on `device`;
        the repack kernels run on that device's current stream."""
        import torch
        device = torch.device(device)
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(device):
            return cls._from_quantized(q, dtype, device)

    @classmethod
    def _from_quantized(cls, q, dtype, device):
        import torch
        from .packing import to_tiles
        oc, ic, k, bits, g = q.oc, q.ic, q.k, q.bits, q.g
        m = ic - k
        m_pad, k_pad = _pad(m, 128), _pad(k, 64)
        widx = np.asarray(q.weak_indices, np.int64)
        p = np.arange(ic) if q.input_perm is None else np.asarray(q.input_perm, np.int64)
        colmap = np.full(m_pad + k_pad, -1, np.int32)
        keep = np.ones(ic, dtype=bool)
        keep[np.asarray(q.weak_indices, np.int64)] = False
        colmap[:m] = p[np.flatnonzero(keep)]
        colmap[m_pad:m_pad + k] = p[widx]
        fast = (q.input_perm is None and q.layout == "structured" and m % 8 == 0 and ic % 8 == 0)
        qweight = to_tiles(q.packed, oc, m, bits, device=device)
        sc = torch.from_numpy(np.ascontiguousarray(q.scales, np.float32)).to(device)
        zr = torch.from_numpy(np.ascontiguousarray(q.zeros, np.float32)).to(device)
        ng = sc.shape[1]
        sz = torch.empty((_pad(oc, 16) * ng * 2,), dtype=torch.float32, device=device)
        L = _lib.lib()
        st = _lib.stream_ptr()
        _lib.check(L.qeft_pack_sz(_lib.ptr(sc), _lib.ptr(zr), oc, ng, _lib.ptr(sz), st), "pack_sz")
        weak32 = torch.from_numpy(np.ascontiguousarray(q.weak, np.float32)).to(device)
        weak16 = torch.empty((_pad(oc, 16), k_pad), dtype=torch_dtype(dtype), device=device)
        if k:
            _lib.check(L.qeft_pack_weak(_lib.ptr(weak32), oc, k, _DT[dtype], _lib.ptr(weak16), st),
                       "pack_weak")
        return cls(oc=oc, ic=ic, k=k, bits=bits, g=g, qweight=qweight, sz=sz, weak16=weak16,
                   colmap=torch.from_numpy(colmap).to(device), dtype=dtype,
                   weak32=weak32.reshape(oc, k), structured_fast=fast, source_id=_source_id(q),
                   sz16=make_sz16(sc, zr, oc, m, g))

    # ------------------------------------------------------------------
    def refresh_weak16(self):
        """Re-pack weak16 from the fp32 master (after an optimizer step)."""
        if self.k:
            _lib.check(_lib.lib().qeft_pack_weak(_lib.ptr(self.weak32), self.oc, self.k,
                                                 _DT[self.dtype], _lib.ptr(self.weak16),
                                                 _lib.stream_ptr()), "pack_weak")

    def dequant_full(self):
        """fp32 [oc][ic] as the kernels see it (fp16/bf16 params, weak16)."""
        import torch
        out = torch.zeros((self.oc, self.ic), dtype=torch.float32, device=self.device)
        _lib.check(_lib.lib().qeft_dequant_full(self.cptr, _lib.ptr(out), _lib.stream_ptr()),
                   "dequant_full")
        return out

    def weight_bytes(self) -> int:
        """Algorithmic HBM bytes one GEMV must read: codes +
        fp16 (scale, zero) pairs (4 B per row and group) + fp16 weak block."""
        from .packing import row_bytes
        return self.oc * row_bytes(self.m, self.bits) + 4 * self.oc * self.ng + 2 * self.oc * self.k

    # ------------------------------------------------------------------
    def gemv(self, x, out=None, out_f32=False, accumulate=False):
        """y[n] = W_hat x[n] for x of shape (n, ic), n <= 16 (decode path). With
        accumulate=True, out += W_hat x in the kernel's epilogue (a fused residual add)."""
        import torch
        _lib.require_cuda(x, "x")
        if x.dim() != 2 or x.shape[1] != self.ic:
            raise ShapeError(f"x shape {tuple(x.shape)} != (n, {self.ic})")
        if x.dtype != self.tdtype:
            raise ShapeError(f"x dtype {x.dtype} != layer dtype {self.tdtype}")
        if x.stride(1) != 1:
            x = x.contiguous()
        n = x.shape[0]
        if out is None:
            if accumulate:
                raise ShapeError("gemv: accumulate needs an output to add to")
            out = torch.empty((n, self.oc), dtype=torch.float32 if out_f32 else self.tdtype,
                              device=x.device)
        L = _lib.lib()
        wsb = int(L.qeft_gemv_workspace_bytes(self.cptr, n))
        ws = GEMV_WORKSPACE.get(wsb, x.device)
        ldx = x.stride(0) if n > 1 else self.ic      # size-1 dims may carry any stride
        ldy = out.stride(0) if n > 1 else self.oc
        if out.stride(1) != 1 or (n > 1 and ldy < self.oc):
            raise ShapeError("gemv: out must be row-major with unit column stride")
        flags = (1 if out.dtype == torch.float32 else 0) | (2 if accumulate else 0)
        _lib.check(L.qeft_gemv(self.cptr, _lib.ptr(x), ldx, _lib.ptr(out), ldy, flags, n, _lib.ptr(ws),
                               ws.numel(), _lib.stream_ptr()), "gemv")
        return out

    def gemv_swiglu(self, g, u, out=None, accumulate=False):
        """y[n] = W_hat (silu(g[n]) * u[n]) (the decode step's down projection, model.py:389-391):
        the SwiGLU runs inside the GEMV's x staging (qeft_gemv_swiglu), bit-identical to
        fused.silu_mul followed by gemv."""
        import torch
        _lib.require_cuda(g, "g")
        if g.shape != u.shape or g.dim() != 2 or g.shape[1] != self.ic or g.dtype != self.tdtype or u.dtype != g.dtype:
            raise ShapeError(f"gemv_swiglu: g {tuple(g.shape)} / u {tuple(u.shape)} incompatible with the layer")
        g, u = g.contiguous(), u.contiguous()
        n = g.shape[0]
        if out is None:
            if accumulate:
                raise ShapeError("gemv_swiglu: accumulate needs an output to add to")
            out = torch.empty((n, self.oc), dtype=self.tdtype, device=g.device)
        L = _lib.lib()
        ws = GEMV_WORKSPACE.get(int(L.qeft_gemv_workspace_bytes(self.cptr, n)), g.device)
        ldy = out.stride(0) if n > 1 else self.oc
        if out.stride(1) != 1 or (n > 1 and ldy < self.oc):
            raise ShapeError("gemv_swiglu: out must be row-major with unit column stride")
        flags = (1 if out.dtype == torch.float32 else 0) | (2 if accumulate else 0)
        _lib.check(L.qeft_gemv_swiglu(self.cptr, _lib.ptr(g), _lib.ptr(u), self.ic, _lib.ptr(out), ldy, flags, n,
                                      _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gemv_swiglu")
        return out

    def gemm_fwd(self, x, out=None):
        """y = x W_hat^T for x of shape (T, ic) (prefill / fine-tune forward)."""
        import torch
        _lib.require_cuda(x, "x")
        if x.dim() != 2 or x.shape[1] != self.ic or x.dtype != self.tdtype:
            raise ShapeError(f"x {tuple(x.shape)} {x.dtype} incompatible with layer")
        if x.stride(1) != 1:
            x = x.contiguous()
        T = x.shape[0]
        if out is None:
            out = torch.empty((T, self.oc), dtype=self.tdtype, device=x.device)
        L = _lib.lib()
        ws = WORKSPACE.get(int(L.qeft_gemm_workspace_bytes(self.cptr, T)), x.device)
        _lib.check(L.qeft_gemm_fwd(self.cptr, _lib.ptr(x), _ld(x), _lib.ptr(out), _ld(out),
                                   T, _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gemm_fwd")
        return out

    def gemm_dgrad(self, dy, out=None, accumulate=False):
        """dx = dy W_hat for dy of shape (T, oc)."""
        import torch
        _lib.require_cuda(dy, "dy")
        if dy.dim() != 2 or dy.shape[1] != self.oc or dy.dtype != self.tdtype:
            raise ShapeError(f"dy {tuple(dy.shape)} {dy.dtype} incompatible with layer")
        if dy.stride(1) != 1:
            dy = dy.contiguous()
        T = dy.shape[0]
        if out is None:
            out = torch.empty((T, self.ic), dtype=self.tdtype, device=dy.device)
            accumulate = False
        L = _lib.lib()
        ws = WORKSPACE.get(int(L.qeft_gemm_workspace_bytes(self.cptr, T)), dy.device)
        _lib.check(L.qeft_gemm_dgrad(self.cptr, _lib.ptr(dy), _ld(dy), _lib.ptr(out),
                                     _ld(out), T, int(accumulate), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_ptr()), "gemm_dgrad")
        return out

    def gather_weak(self, x, out=None):
        """x_weak[t][j] = x[t][weak_j] (T x roundup(k, 8), zero padded): the only slice of the
        input the weak-column backward needs (TrainableLayerState.x_weak, tuning.py:30-34)."""
        import torch
        kw = _pad(self.k, 8)
        if x.stride(1) != 1:
            x = x.contiguous()
        T = x.shape[0]
        if out is None:
            out = torch.empty((T, kw), dtype=x.dtype, device=x.device)
        if self.k:
            _lib.check(_lib.lib().qeft_gather_cols(
                _lib.ptr(x), _ld(x), self.colmap.data_ptr() + 4 * self.m_pad, kw, T,
                _DT[self.dtype], _lib.ptr(out), _lib.stream_ptr()), "gather_weak")
        return out

    def gemm_wgrad_weak(self, dy, x_weak, out=None, accumulate=False):
        """dW_weak[o][j] (+)= sum_t dy[t][o] x_weak[t][j], fp32 (oc, k) from the saved slice."""
        import torch
        if dy.stride(1) != 1:
            dy = dy.contiguous()
        T = dy.shape[0]
        if out is None:
            out = torch.empty((self.oc, self.k), dtype=torch.float32, device=dy.device)
            accumulate = False
        if not self.k:
            return out
        L = _lib.lib()
        ws = WORKSPACE.get(int(L.qeft_gemm_workspace_bytes(self.cptr, T)), dy.device)
        _lib.check(L.qeft_gemm_wgrad_weak(self.cptr, _lib.ptr(dy), _ld(dy), _lib.ptr(x_weak),
                                          _ld(x_weak), _lib.ptr(out), T, int(accumulate),
                                          _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gemm_wgrad_weak")
        return out

    def gemm_wgrad(self, dy, x, out=None, accumulate=False):
        """dW_weak[o][j] = sum_t dy[t][o] x[t][weak_j], fp32 (oc, k)."""
        import torch
        if dy.stride(1) != 1:
            dy = dy.contiguous()
        if x.stride(1) != 1:
            x = x.contiguous()
        T = dy.shape[0]
        if out is None:
            out = torch.empty((self.oc, self.k), dtype=torch.float32, device=dy.device)
            accumulate = False
        L = _lib.lib()
        ws = WORKSPACE.get(int(L.qeft_gemm_workspace_bytes(self.cptr, T)), dy.device)
        _lib.check(L.qeft_gemm_wgrad(self.cptr, _lib.ptr(dy), _ld(dy), _lib.ptr(x), _ld(x),
                                     _lib.ptr(out), T, int(accumulate), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_ptr()), "gemm_wgrad")
        return out


def _ld(t) -> int:
    """Row pitch of a row-major 2-D tensor; a single row may carry any stride(0)."""
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


def _source_id(q):
    """Identity of the frozen parts of a host record the device copy was built from: the
    packed codes, the (scale, zero) arrays, the weak column set and the input permutation.
    The trainable weak block is NOT part of it: `device_layer` re-syncs it by content."""
    perm = getattr(q, "input_perm", None)
    return (id(q.packed), id(q.scales), id(q.zeros), q.layout,
            np.asarray(q.weak_indices, np.int64).tobytes(),
            None if perm is None else np.asarray(perm, np.int64).tobytes())


class _DeviceCache:
    """Device copies of host QuantizedLinear records, keyed by the record itself.

    The reference's records (pkg/src/qeft/quantizer.py:42-57) are plain dataclasses with no
    room for a device handle, and its fine-tune loop updates `q.weak` IN PLACE between steps
    (tuning.py:159 adam_step, 234-236). So the cache lives here, not on the record: an entry
    is dropped when its record is garbage collected (weakref finalizer), rebuilt when a frozen
    field is replaced, and its weak block is re-uploaded whenever the host `q.weak` bytes
    differ from the last upload (a memcmp of oc x k floats per call -- the reference itself
    reads q.weak live on every call)."""

    def __init__(self):
        self.entries = {}  # (id(record), dtype, device) -> [weakref, source_id, weak snapshot, DeviceLayer]

    def get(self, q, dtype="f16", device=None):
        import torch
        import weakref
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        key = (id(q), dtype, str(dev))
        e = self.entries.get(key)
        sid = _source_id(q)
        if e is None or e[0]() is not q or e[1] != sid:
            with torch.cuda.device(dev):
                dl = DeviceLayer.from_quantized(q, dtype=dtype, device=dev)
            try:
                ref = weakref.ref(q, lambda _r, k=key: self.entries.pop(k, None))
            except TypeError:  # records without weakref support stay cached until replaced
                ref = (lambda obj=q: obj)
            e = [ref, sid, np.array(q.weak, np.float32, copy=True), dl]
            self.entries[key] = e
        elif q.k and not np.array_equal(e[2], q.weak):
            dl = e[3]
            dl.weak32.copy_(torch.from_numpy(np.ascontiguousarray(q.weak, np.float32)))
            with torch.cuda.device(dev):
                dl.refresh_weak16()
            e[2] = np.array(q.weak, np.float32, copy=True)
        return e[3]


DEVICE_CACHE = _DeviceCache()


def device_layer(q, dtype: str = "f16", device=None) -> DeviceLayer:
    """The B200 tile-layout copy of a host QuantizedLinear (ours or the reference's own
    record class), cached per (record, dtype, device) with its weak block kept in sync."""
    return DEVICE_CACHE.get(q, dtype, device)
