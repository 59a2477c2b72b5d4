"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 QEFT linear-layer path. It is a
numpy restatement of the reference package's algorithms (arXiv 2410.08661,
`/root/reference/pkg/src/qeft`), written independently from the reference
source and citing the file:line of every behaviour it restates.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import it. The product package
(`paper_2410_08661_b200`) never imports it; the product path runs the CUDA
library and fails loudly when it is missing.

Parity is pinned: `tests/test_oracle_golden.py` checks every function here
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py` imports `/root/reference/pkg/src/qeft` and
writes `tests/golden/*.npz`), plus the known-answer vectors from the
reference's own unit tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class OracleShapeError(ValueError):
    """Mirrors qeft.errors.ShapeError (errors.py:16-17)."""


# ---------------------------------------------------------------------------
# packing  (packing.py:15-72)

def row_bytes(m: int, bits: int) -> int:
    # packing.py:15-21: 4-bit two codes per byte, 3-bit bitstream padded to a byte
    if bits == 4:
        return (m + 1) // 2
    if bits == 3:
        return (3 * m + 7) // 8
    raise OracleShapeError(f"bits={bits}")


def pack_codes(codes, bits: int) -> bytes:
    """packing.py:24-52. Row-major; LSB-first bit order inside every byte."""
    c = np.asarray(codes)
    if c.ndim != 2:
        raise OracleShapeError("codes must be 2-D")
    if bits not in (3, 4):
        raise OracleShapeError(f"bits={bits}")
    if c.size and (c.min() < 0 or c.max() > (1 << bits) - 1):
        raise OracleShapeError("code out of range")
    oc, m = c.shape
    rb = row_bytes(m, bits)
    # code j occupies stream bits [bits*j, bits*j + bits) of its row (for 4-bit
    # this is "even column in the low nibble", packing.py:38-39)
    stream = ((c.astype(np.uint8)[:, :, None] >> np.arange(bits, dtype=np.uint8)) & 1)
    stream = np.concatenate([stream.reshape(oc, bits * m),
                             np.zeros((oc, 8 * rb - bits * m), np.uint8)], axis=1)
    weights = (1 << np.arange(8, dtype=np.uint32))
    return (stream.reshape(oc, rb, 8).astype(np.uint32) @ weights).astype(np.uint8).tobytes()


def unpack_codes(data: bytes, oc: int, m: int, bits: int) -> np.ndarray:
    """packing.py:55-72 (inverse of pack_codes)."""
    rb = row_bytes(m, bits)
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    if raw.size != oc * rb:
        raise OracleShapeError("payload size mismatch")
    raw = raw.reshape(oc, rb)
    if bits == 4:  # nibble split: low nibble = even column
        return np.ascontiguousarray(np.stack([raw & 15, raw >> 4], axis=2).reshape(oc, 2 * rb)[:, :m])
    fields = np.unpackbits(raw, axis=1, bitorder="little")[:, :3 * m].reshape(oc, m, 3)
    return fields[:, :, 0] | (fields[:, :, 1] << 1) | (fields[:, :, 2] << 2)


# ---------------------------------------------------------------------------
# groups  (quantizer.py:103-109, 83-84)

def n_groups(m: int, g: int) -> int:
    return max(1, math.ceil(m / g)) if m > 0 else 0


def group_bounds(m: int, g: int):
    return [(s, min(s + g, m)) for s in range(0, m, g)]


# ---------------------------------------------------------------------------
# per-group parameter search  (quantizer.py:115-218)

def minmax_scale_zero(seg, bits: int):
    """quantizer.py:115-120: min-max, constant group -> (1, wmin)."""
    lo, hi = float(np.min(seg)), float(np.max(seg))
    if lo == hi:
        return 1.0, lo
    return (hi - lo) / (2 ** bits - 1), lo


def grid_scale_zero(seg, bits: int, steps: int = 100, amin: float = 0.5):
    """quantizer.py:144-179: shrink [min,max] about the midpoint by alpha,
    keep the alpha with least fp64 squared error, larger alpha on ties."""
    w = np.asarray(seg, dtype=np.float64)
    if steps < 1:
        raise OracleShapeError("grid_steps must be >= 1")
    lo0, hi0 = float(w.min()), float(w.max())
    if lo0 == hi0:
        return 1.0, lo0
    alphas = [1.0] if steps == 1 else list(
        amin + np.arange(steps) * (1.0 - amin) / (steps - 1))
    mid = 0.5 * (lo0 + hi0)
    levels = 2 ** bits - 1
    best_err, best = None, None
    for a in alphas:
        if a == 1.0:
            lo, hi = lo0, hi0
        else:
            lo, hi = mid - a * (mid - lo0), mid + a * (hi0 - mid)
        s = (hi - lo) / levels
        c = np.clip(np.rint((w - lo) / s), 0, levels)
        e = float(np.sum((w - (c * s + lo)) ** 2))
        if best_err is None or e <= best_err:
            best_err, best = e, (s, lo)
    return best


def layer_params(wd, bits: int, g: int, mode: str, steps=100, amin=0.5):
    """quantizer.py:191-208: per (row, group) params, stored float32."""
    oc, m = wd.shape
    ng = n_groups(m, g)
    sc = np.empty((oc, ng), np.float32)
    zr = np.empty((oc, ng), np.float32)
    for gi, (a, b) in enumerate(group_bounds(m, g)):
        for r in range(oc):
            if mode == "rtn":
                s, z = minmax_scale_zero(wd[r, a:b], bits)
            else:
                s, z = grid_scale_zero(wd[r, a:b], bits, steps, amin)
            sc[r, gi], zr[r, gi] = s, z
    return sc, zr


def nearest_codes(wd, sc, zr, g: int, bits: int):
    """quantizer.py:211-218: clip(rint((w64 - z)/s)) per group."""
    oc, m = wd.shape
    out = np.empty((oc, m), np.uint8)
    for gi, (a, b) in enumerate(group_bounds(m, g)):
        q = np.rint((wd[:, a:b].astype(np.float64) - zr[:, gi:gi + 1]) / sc[:, gi:gi + 1])
        out[:, a:b] = np.clip(q, 0, 2 ** bits - 1).astype(np.uint8)
    return out


def optq_codes(wd, h, sc, zr, g: int, bits: int):
    """quantizer.py:221-259: greedy column rounding with inverse-Hessian
    error feedback (1% mean-diagonal damping, upper Cholesky of H^-1);
    nearest-rounding fallback when the damped Hessian is not factorizable."""
    w = np.array(wd, dtype=np.float64)
    oc, m = w.shape
    if h.shape != (m, m):
        raise OracleShapeError("Hessian shape")
    hd = np.array(h, dtype=np.float64)
    hd[np.diag_indices(m)] += 0.01 * float(np.mean(np.diagonal(hd)))
    try:
        u = np.linalg.cholesky(np.linalg.inv(hd)).T
    except np.linalg.LinAlgError:
        return nearest_codes(wd, sc, zr, g, bits), True
    lv = 2 ** bits - 1
    s64, z64 = sc.astype(np.float64), zr.astype(np.float64)
    ng = s64.shape[1]
    out = np.empty((oc, m), np.uint8)
    for i in range(m):
        gi = min(i // g, ng - 1)
        col = w[:, i]
        q = np.clip(np.rint((col - z64[:, gi]) / s64[:, gi]), 0, lv)
        out[:, i] = q.astype(np.uint8)
        e = (col - (q * s64[:, gi] + z64[:, gi])) / u[i, i]
        if i + 1 < m:
            w[:, i + 1:] -= np.outer(e, u[i, i + 1:])
    return out, False


# ---------------------------------------------------------------------------
# the quantized-layer record and quantize_layer  (quantizer.py:42-100, 265-344)

@dataclass
class OracleLayer:
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
    def m(self):
        return self.ic - self.k

    @property
    def n_groups(self):
        return n_groups(self.m, self.g)

    def codes(self):
        return unpack_codes(self.packed, self.oc, self.m, self.bits)

    def quant_positions(self):
        keep = np.ones(self.ic, bool)
        keep[self.weak_indices] = False
        return np.flatnonzero(keep)

    def dequant_dense(self):
        # quantizer.py:87-93: f32(code) * scale + zero, f32 multiply then add
        c = self.codes().astype(np.float32)
        out = np.empty_like(c)
        for gi, (a, b) in enumerate(group_bounds(self.m, self.g)):
            out[:, a:b] = c[:, a:b] * self.scales[:, gi:gi + 1] + self.zeros[:, gi:gi + 1]
        return out

    def dequant_full(self):
        # quantizer.py:95-100
        full = np.empty((self.oc, self.ic), np.float32)
        full[:, self.quant_positions()] = self.dequant_dense()
        full[:, self.weak_indices] = self.weak
        return full


def topk_ascending(scores, k: int):
    """calibration.py:135-143: stable argsort of -score, first k, sorted."""
    s = np.asarray(scores)
    if k > s.shape[0]:
        raise OracleShapeError("k too large")
    if k == 0:
        return np.zeros(0, np.int64)
    return np.sort(np.argsort(-s, kind="stable")[:k]).astype(np.int64)


def quantize_layer(w, *, k, bits, g, mode="optq", layout="structured",
                   lam=None, indices=None, x=None, h=None,
                   grid_steps=100, alpha_min=0.5) -> OracleLayer:
    """quantizer.py:265-344."""
    w = np.asarray(w, np.float32)
    oc, ic = w.shape
    if k >= ic:
        raise OracleShapeError("k must be < IC")
    if bits not in (3, 4):
        raise OracleShapeError("bits")
    if mode not in ("optq", "rtn"):
        raise OracleShapeError("mode")
    if layout == "structured":
        widx = np.arange(ic - k, ic, dtype=np.int64)
        if indices is not None and not np.array_equal(np.sort(np.asarray(indices)), widx):
            raise OracleShapeError("structured needs trailing weak columns")
    elif layout == "irregular":
        if indices is None:
            if lam is None:
                raise OracleShapeError("irregular needs indices or lambda")
            widx = topk_ascending(lam, k)
        else:
            widx = np.sort(np.asarray(indices, np.int64))
            if widx.size != k or (widx.size and (widx[0] < 0 or widx[-1] >= ic)):
                raise OracleShapeError("weak index set invalid")
            if np.unique(widx).size != widx.size:
                raise OracleShapeError("duplicate weak indices")
    else:
        raise OracleShapeError("layout")
    keep = np.ones(ic, bool)
    keep[widx] = False
    qpos = np.flatnonzero(keep)
    wd = w[:, qpos]
    m = wd.shape[1]
    geff = min(g, m) if m else g
    sc, zr = layer_params(wd, bits, geff, "rtn" if mode == "rtn" else "grid",
                          grid_steps, alpha_min)
    fb = False
    if mode == "optq" and m > 0:
        if h is None:
            if x is None:
                raise OracleShapeError("optq needs x or h")
            xs = np.asarray(x, np.float64)
            if xs.shape[0] != ic:
                raise OracleShapeError("calibration rows")
            h = 2.0 * xs @ xs.T
        hq = np.asarray(h, np.float64)[np.ix_(qpos, qpos)]
        codes, fb = optq_codes(wd, hq, sc, zr, geff, bits)
    else:
        codes = nearest_codes(wd, sc, zr, geff, bits)
    return OracleLayer(oc=oc, ic=ic, k=k, bits=bits, g=geff,
                       packed=pack_codes(codes, bits), scales=sc, zeros=zr,
                       weak=np.ascontiguousarray(w[:, widx]), weak_indices=widx,
                       layout=layout, mode=mode, optq_fallback=fb)


# ---------------------------------------------------------------------------
# matvec paths  (kernels.py:54-157)

def analytic_bytes(q) -> int:
    # kernels.py:54-58 (reference accounting: fp32 params + fp32 weak)
    return len(q.packed) + 8 * q.oc * q.n_groups + 4 * q.oc * q.k


def analytic_fmas(q) -> int:
    # kernels.py:61-63
    return q.oc * q.m + 2 * q.oc * q.n_groups + q.oc * q.k


def grouped_fold(q, xq, xw):
    """kernels.py:66-75: y = sum_g s_g*(c_g . x_g) + z_g*sum(x_g) + weak . x_w."""
    c = q.codes().astype(np.float32)
    y = np.zeros(q.oc, np.float32)
    for gi, (a, b) in enumerate(group_bounds(q.m, q.g)):
        y += q.scales[:, gi] * (c[:, a:b] @ xq[a:b]) + q.zeros[:, gi] * np.float32(xq[a:b].sum())
    if q.k:
        y += q.weak @ xw
    return y


def matvec_structured(q, x):
    # kernels.py:87-98
    if q.layout != "structured":
        raise OracleShapeError("layout")
    x = np.asarray(x, np.float32)
    if x.shape != (q.ic,):
        raise OracleShapeError("x shape")
    return grouped_fold(q, x[:q.m], x[q.m:])


def matvec_irregular(q, x):
    # kernels.py:101-112
    if q.layout != "irregular":
        raise OracleShapeError("layout")
    x = np.asarray(x, np.float32)
    if x.shape != (q.ic,):
        raise OracleShapeError("x shape")
    return grouped_fold(q, x[q.quant_positions()], x[q.weak_indices])


def matvec_online_reorder(q, x, perm):
    # kernels.py:115-126
    p = np.asarray(getattr(perm, "perm", perm), np.int64)
    if p.shape != (q.ic,):
        raise OracleShapeError("perm")
    x = np.asarray(x, np.float32)
    return grouped_fold(q, x[p[:q.m]], x[p[q.m:]])


def matvec_reference(q, x):
    # kernels.py:129-134: float64 dense oracle
    x = np.asarray(x, np.float64)
    if q.input_perm is not None:
        x = x[q.input_perm]
    return q.dequant_full().astype(np.float64) @ x


def matvec_native(q, x):
    # kernels.py:137-157 (native_path order: online, structured, irregular)
    if q.input_perm is not None:
        return matvec_online_reorder(q, x, q.input_perm)
    if q.layout == "structured":
        return matvec_structured(q, x)
    return matvec_irregular(q, x)


# ---------------------------------------------------------------------------
# weak-only training forward / backward  (tuning.py:52-103)

def forward_train(q, x):
    """tuning.py:52-72: Y = W_full @ X, keep X[weak] (k x T)."""
    x = np.asarray(x, np.float32)
    if x.shape[0] != q.ic:
        raise OracleShapeError("input rows")
    if q.input_perm is not None:
        x = x[q.input_perm]
    y = q.dequant_full() @ x
    return y, np.ascontiguousarray(x[q.weak_indices])


def backward(q, x_weak, dy):
    """tuning.py:75-103: dX through the full matrix, dW for weak columns only."""
    dy = np.asarray(dy, np.float32)
    if dy.shape != (q.oc, x_weak.shape[1]):
        raise OracleShapeError("dY shape")
    dx = q.dequant_full().T @ dy
    if q.input_perm is not None:
        out = np.empty_like(dx)
        out[q.input_perm] = dx
        dx = out
    return dx, dy @ x_weak.T


def cost_counters(q, t: int):
    # tuning.py:99-102
    return dict(wgrad_fma=q.oc * q.k * t, full_fma=q.oc * q.ic * t,
                saved_elems=q.k * t, full_elems=q.ic * t)


# ---------------------------------------------------------------------------
# optimizer  (tuning.py:137-160, 226-236)

@dataclass
class AdamMoments:
    m: np.ndarray
    v: np.ndarray
    step: int = 0


def adam_update(st: AdamMoments, w, grad, lr, b1=0.9, b2=0.999, eps=1e-8):
    """tuning.py:148-160, in place on w (float32 moments, fp64 bias terms)."""
    if not np.all(np.isfinite(grad)):
        raise FloatingPointError("non-finite gradient")
    st.step += 1
    st.m = b1 * st.m + (1.0 - b1) * grad
    st.v = b2 * st.v + (1.0 - b2) * grad * grad
    mh = st.m / (1.0 - b1 ** st.step)
    vh = st.v / (1.0 - b2 ** st.step)
    w -= (lr * mh / (np.sqrt(vh) + eps)).astype(w.dtype)
    return w


def clip_scale(grads, max_norm):
    """tuning.py:226-233: global fp64 L2 norm; scale only when above max."""
    gn = math.sqrt(sum(float(np.sum(np.asarray(g, np.float64) ** 2)) for g in grads))
    sc = 1.0
    if max_norm and gn > max_norm:
        sc = max_norm / (gn + 1e-12)
    return gn, sc


# ---------------------------------------------------------------------------
# weak-column selection and reordering  (calibration.py:73-187, reorder.py:56-63)

def lambda_running(prev, n, x):
    """calibration.py:73-98: running mean over sequences of 2*sum_t X^2."""
    c = 2.0 * np.sum(np.asarray(x, np.float64) ** 2, axis=1)
    if prev is None:
        return c, 1
    return (prev * n + c) / (n + 1), n + 1


RESID_SUFFIXES = ("wq", "wk", "wv", "w_up", "w_gate")


def select_global(lam: dict, k: int, n_blocks: int):
    """calibration.py:146-187. Returns (resid, ffn list, wo list, s_global)."""
    resid_names = [n for n in lam if n == "head" or n.split(".")[-1] in RESID_SUFFIXES]
    if not resid_names:
        raise OracleShapeError("no residual-fed layers")
    d = lam[resid_names[0]].shape[0]
    s = np.zeros(d, np.float64)
    for n in resid_names:
        v = lam[n].astype(np.float64)
        if v.shape[0] != d:
            raise OracleShapeError("IC mismatch")
        ids = topk_ascending(v, k)
        mu = v.mean()
        if mu > 0:
            s[ids] += v[ids] / mu
    ffn = [topk_ascending(lam[f"b{i}.w_down"], k) for i in range(n_blocks)]
    wo = [topk_ascending(lam[f"b{i}.wo"], k) for i in range(n_blocks)]
    return topk_ascending(s, k), ffn, wo, s


def weak_to_tail(n: int, weak) -> np.ndarray:
    """reorder.py:56-63: perm[new] = old = [ascending non-weak, ascending weak]."""
    w = np.sort(np.asarray(weak, np.int64))
    if w.size and (w[0] < 0 or w[-1] >= n):
        raise OracleShapeError("weak index out of range")
    mask = np.zeros(n, bool)
    mask[w] = True
    return np.concatenate([np.flatnonzero(~mask), w]).astype(np.int64)
