"""The QuantizedLinear record and `quantize_layer` (reference API).

Mirrors pkg/src/qeft/quantizer.py: the record keeps the reference fields and
byte format (so it interchanges with the reference's containers and tests);
`quantize_layer` runs on the GPU:
  * mode="rtn": min-max params + nearest codes in one CUDA kernel
    (libqeft_b200 `qeft_quantize_rtn`), bit-exact with quantizer.py:115-120,
    211-218;
  * mode="optq": the alpha-grid parameter search (quantizer.py:144-179, CUDA kernel,
    bit-exact) and the OPTQ column loop with inverse-Hessian error feedback
    (quantizer.py:221-259): H = 2 X X^T (fp64 GEMM on the GPU when X is given), the factor
    U = chol(inv(H + damping))^T in fp64 on the GPU (cuSOLVER via torch.linalg; set
    QEFT_OPTQ_FACTOR=host for the reference's own LAPACK factor), and the O(oc m^2) sweep in
    the `qeft_optq_codes` kernel, bit-exact given the factor. Codes match the reference
    except where the LAPACK vs cuSOLVER rounding of the factor moves a value across a
    rounding boundary.
Weak-column selection (irregular layouts) reuses calibration.select_local_topk
and is bit-exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError
from .packing import pack_codes, unpack_codes

LAYOUT_STRUCTURED = "structured"
LAYOUT_IRREGULAR = "irregular"
GRID_STEPS_DEFAULT = 100
ALPHA_MIN_DEFAULT = 0.5
OPTQ_DAMP_FRAC = 0.01


def _n_groups(m: int, g: int) -> int:
    return max(1, math.ceil(m / g)) if m > 0 else 0


def group_slices(m: int, g: int):
    """(start, stop) per group along the m quantized columns; last may be ragged
    (quantizer.py:107-109)."""
    return [(lo, min(lo + g, m)) for lo in range(0, m, g)]


@dataclass
class QuantizedLinear:
    """Same fields and meaning as the reference record (quantizer.py:42-57)."""
    oc: int
    ic: int
    k: int
    bits: int
    g: int
    packed: bytes
    scales: np.ndarray
    zeros: np.ndarray
    weak: np.ndarray
    weak_indices: np.ndarray
    layout: str
    mode: str = "optq"
    optq_fallback: bool = False
    input_perm: np.ndarray | None = None

    @property
    def m(self) -> int:
        return self.ic - self.k

    @property
    def n_groups(self) -> int:
        return _n_groups(self.m, self.g)

    def codes(self) -> np.ndarray:
        return unpack_codes(self.packed, self.oc, self.m, self.bits)

    def quant_positions(self) -> np.ndarray:
        keep = np.ones(self.ic, dtype=bool)
        keep[self.weak_indices] = False
        return np.flatnonzero(keep)

    def group_of(self, col: int) -> int:
        return min(col // self.g, self.n_groups - 1) if self.m else 0

    def dequant_dense(self) -> np.ndarray:
        """Host view of the dequantized (oc, m) part, f32(code)*scale + zero
        (quantizer.py:87-93); a format accessor, not the compute path."""
        c = self.codes().astype(np.float32)
        gidx = np.minimum(np.arange(self.m) // self.g, max(self.n_groups - 1, 0))
        return c * self.scales[:, gidx] + self.zeros[:, gidx]

    def dequant_full(self) -> np.ndarray:
        out = np.empty((self.oc, self.ic), dtype=np.float32)
        out[:, self.quant_positions()] = self.dequant_dense()
        out[:, self.weak_indices] = self.weak
        return out

    # --- B200 device copy -------------------------------------------------
    def device(self, dtype="f16"):
        """The B200 tile-layout copy on the current CUDA device (layer.device_layer: cached
        per record, weak block re-synced from self.weak when it changes)."""
        from .layer import device_layer
        return device_layer(self, dtype)


# ---------------------------------------------------------------------------

def _select_weak(ic, k, layout, lam, indices):
    if layout == LAYOUT_STRUCTURED:
        trailing = np.arange(ic - k, ic, dtype=np.int64)
        if indices is not None and not np.array_equal(np.sort(np.asarray(indices)), trailing):
            raise ShapeError("structured layout requires trailing weak columns")
        return trailing
    if layout == LAYOUT_IRREGULAR:
        if indices is None:
            if lam is None:
                raise ShapeError("irregular layout needs indices or lambda")
            from .calibration import select_local_topk
            return select_local_topk(np.asarray(lam), k)
        widx = np.sort(np.asarray(indices, dtype=np.int64))
        if widx.size != k or (widx.size and (widx[0] < 0 or widx[-1] >= ic)):
            raise ShapeError("weak index set invalid for layer")
        if np.unique(widx).size != widx.size:
            raise ShapeError("duplicate weak indices")
        return widx
    raise ShapeError(f"unknown layout {layout!r}")


def _rtn_gpu(w_dense: np.ndarray, g: int, bits: int):
    import torch
    oc, m = w_dense.shape
    ng = _n_groups(m, g)
    wd = torch.from_numpy(np.ascontiguousarray(w_dense, np.float32)).cuda()
    sc = torch.empty((oc, ng), dtype=torch.float32, device="cuda")
    zr = torch.empty_like(sc)
    codes = torch.empty((oc, m), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().qeft_quantize_rtn(_lib.ptr(wd), oc, m, g, bits, _lib.ptr(sc), _lib.ptr(zr),
                                            _lib.ptr(codes), _lib.stream_ptr()), "quantize_rtn")
    return sc.cpu().numpy(), zr.cpu().numpy(), codes.cpu().numpy()


def _grid_params_gpu(w_dense: np.ndarray, g: int, bits: int, steps: int, amin: float):
    """alpha-grid search (quantizer.py:144-179) for every (row, group): libqeft_b200
    `qeft_grid_params`, bit-exact with the reference (fp64 op order, numpy pairwise sums)."""
    import torch
    if steps < 1:
        raise ShapeError("grid_steps must be >= 1")
    oc, m = w_dense.shape
    ng = _n_groups(m, g)
    wd = torch.from_numpy(np.ascontiguousarray(w_dense, np.float32)).cuda()
    sc = torch.empty((oc, ng), dtype=torch.float32, device="cuda")
    zr = torch.empty_like(sc)
    _lib.check(_lib.lib().qeft_grid_params(_lib.ptr(wd), oc, m, g, bits, int(steps), float(amin),
                                           _lib.ptr(sc), _lib.ptr(zr), _lib.stream_ptr()), "grid_params")
    return sc.cpu().numpy(), zr.cpu().numpy()


def _optq_factor(h):
    """U = chol(inv(H + 1% mean-diag damping)).T exactly as the reference computes it on the host
    (quantizer.py:236-242); None where the reference falls back (LinAlgError)."""
    hd = np.asarray(h, dtype=np.float64).copy()
    m = hd.shape[0]
    damp = OPTQ_DAMP_FRAC * float(np.mean(np.diagonal(hd)))
    hd[np.diag_indices(m)] += damp
    try:
        hinv = np.linalg.inv(hd)
        return np.ascontiguousarray(np.linalg.cholesky(hinv).T)
    except np.linalg.LinAlgError:
        return None


def _optq_factor_device(h):
    """The same factor in fp64 on the GPU (cuSOLVER getrf/getri + potrf through torch.linalg);
    None where the reference would fall back (singular H or a non-positive-definite inverse)."""
    import torch
    hd = h.to(torch.float64).clone()
    damp = OPTQ_DAMP_FRAC * float(hd.diagonal().mean())
    hd.diagonal().add_(damp)
    hinv, info = torch.linalg.inv_ex(hd)
    if int(info) != 0 or not bool(torch.isfinite(hinv).all()):
        return None
    lo, info = torch.linalg.cholesky_ex(hinv)
    if int(info) != 0:
        return None
    return lo.T.contiguous()


def optq_factor_mode() -> str:
    import os
    return os.environ.get("QEFT_OPTQ_FACTOR", "device")


def _optq_gpu(w_dense, h, sc, zr, g, bits):
    """Greedy OPTQ rounding (quantizer.py:221-259): factor on the GPU (or the host LAPACK one,
    QEFT_OPTQ_FACTOR=host), then the O(oc*m^2) column sweep in libqeft_b200 (`qeft_optq_codes`),
    bit-exact given the factor."""
    import torch
    if optq_factor_mode() == "host":
        u = _optq_factor(h.cpu().numpy() if hasattr(h, "is_cuda") else h)
        ud = None if u is None else torch.from_numpy(u).cuda()
    else:
        hd = h if hasattr(h, "is_cuda") else torch.from_numpy(np.ascontiguousarray(h, np.float64)).cuda()
        ud = _optq_factor_device(hd)
    if ud is None:
        return None
    oc, m = w_dense.shape
    w = torch.from_numpy(np.array(w_dense, np.float64)).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sc, np.float32)).cuda()
    z = torch.from_numpy(np.ascontiguousarray(zr, np.float32)).cuda()
    err = torch.empty((oc, m), dtype=torch.float64, device="cuda")
    codes = torch.empty((oc, m), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().qeft_optq_codes(_lib.ptr(w), _lib.ptr(ud), _lib.ptr(s), _lib.ptr(z), oc, m, g, bits,
                                          _lib.ptr(err), _lib.ptr(codes), _lib.stream_ptr()), "optq_codes")
    return codes.cpu().numpy()


def _nearest_codes_gpu(w_dense, sc, zr, g, bits):
    """Independent nearest rounding on fixed params (quantizer.py:211-218): `qeft_nearest_codes`."""
    import torch
    oc, m = w_dense.shape
    wd = torch.from_numpy(np.ascontiguousarray(w_dense, np.float32)).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sc, np.float32)).cuda()
    z = torch.from_numpy(np.ascontiguousarray(zr, np.float32)).cuda()
    codes = torch.empty((oc, m), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().qeft_nearest_codes(_lib.ptr(wd), oc, m, g, bits, _lib.ptr(s), _lib.ptr(z),
                                             _lib.ptr(codes), _lib.stream_ptr()), "nearest_codes")
    return codes.cpu().numpy()


def quantize_layer(w, *, k: int, bits: int, g: int, mode: str = "optq",
                   layout: str = LAYOUT_STRUCTURED, lam=None, indices=None, x=None, h=None,
                   grid_steps: int = GRID_STEPS_DEFAULT,
                   alpha_min: float = ALPHA_MIN_DEFAULT) -> QuantizedLinear:
    """Quantize one weight matrix into the mixed-precision layout
    (reference signature and validation, quantizer.py:265-344)."""
    w = np.asarray(w, dtype=np.float32)
    oc, ic = w.shape
    if k >= ic:
        raise ShapeError(f"k={k} must be < IC={ic}")
    if bits not in (3, 4):
        raise ShapeError(f"bits must be 3 or 4, got {bits}")
    if mode not in ("optq", "rtn"):
        raise ShapeError(f"unknown mode {mode!r}")
    widx = _select_weak(ic, k, layout, lam, indices)
    keep = np.ones(ic, dtype=bool)
    keep[widx] = False
    qpos = np.flatnonzero(keep)
    w_dense = np.ascontiguousarray(w[:, qpos])
    m = w_dense.shape[1]
    g_eff = min(g, m) if m else g
    fallback = False
    if mode == "rtn":
        scales, zeros, codes = _rtn_gpu(w_dense, g_eff, bits)
    else:
        scales, zeros = _grid_params_gpu(w_dense, g_eff, bits, grid_steps, alpha_min)
        if m > 0:
            import torch
            if h is None:
                if x is None:
                    raise ShapeError("optq mode needs calibration x or h")
                xs = (x if hasattr(x, "is_cuda") else torch.from_numpy(np.asarray(x, np.float64))).cuda().double()
                if xs.shape[0] != ic:
                    raise ShapeError(f"calibration rows {xs.shape[0]} != IC {ic}")
                h = torch.matmul(xs, xs.T).mul_(2.0)  # quantizer.py:324-332, fp64 GEMM on the GPU
            if hasattr(h, "is_cuda"):
                qi = torch.from_numpy(qpos).to(h.device)
                hq = h.double().index_select(0, qi).index_select(1, qi)
            else:
                hq = np.asarray(h, dtype=np.float64)[np.ix_(qpos, qpos)]
            if tuple(hq.shape) != (m, m):
                raise ShapeError(f"Hessian {tuple(hq.shape)} does not match {m} columns")
            codes = _optq_gpu(w_dense, hq, scales, zeros, g_eff, bits)
            if codes is None:
                codes, fallback = _nearest_codes_gpu(w_dense, scales, zeros, g_eff, bits), True
        else:
            codes = np.zeros((oc, 0), np.uint8)
    return QuantizedLinear(
        oc=oc, ic=ic, k=k, bits=bits, g=g_eff, packed=pack_codes(codes, bits),
        scales=scales, zeros=zeros, weak=np.ascontiguousarray(w[:, widx]),
        weak_indices=widx, layout=layout, mode=mode, optq_fallback=fallback)
