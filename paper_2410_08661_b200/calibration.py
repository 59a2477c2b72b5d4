"""Calibration statistics and weak-column selection.

* HessianFull / accumulate_hessian_full (calibration.py:101-122): the per-layer running mean
  of 2 X X^T over calibration sequences, the input of OPTQ error compensation. Computed on
  the GPU: X^T X is a plain fp64 GEMM (cuBLAS DGEMM through torch -- products of fp32 values
  are exact in fp64, so only the summation order differs from the reference's BLAS call),
  and the running mean is updated in place on the device, (prev * n + c) / (n + 1) in fp64.
* selection (calibration.py:73-187): host-side integer work with identical numpy semantics
  (stable argsort, lower index wins ties, fp64 score accumulation in trace order); it runs
  once per model offline, so there is nothing there worth a kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ShapeError

RESID_SUFFIXES = ("wq", "wk", "wv", "w_up", "w_gate")
HEAD_NAME = "head"


@dataclass
class HessianDiag:
    """Per-layer lambda = running mean of 2*sum_t X^2 (calibration.py:60-64)."""
    lam: dict
    sample_count: int = 0


@dataclass
class HessianFull:
    """calibration.py:101-110: full 2 X X^T running means per layer (name -> IC x IC fp64,
    CUDA tensors; `numpy()` gives the host dict), in trace (insertion) order."""
    h: dict
    sample_count: int = 0

    def diag(self) -> HessianDiag:
        """lambda = the diagonals (calibration.py:107-110), as host fp64 arrays."""
        return HessianDiag(lam={k: _host(v).diagonal().copy() if not hasattr(v, "is_cuda")
                                else v.diagonal().cpu().numpy().copy() for k, v in self.h.items()},
                           sample_count=self.sample_count)

    def numpy(self) -> dict:
        return {k: _host(v) for k, v in self.h.items()}


def _host(v):
    return v.cpu().numpy() if hasattr(v, "is_cuda") else np.asarray(v, np.float64)


def accumulate_hessian_full(trace, running: HessianFull | None = None, device=None) -> HessianFull:
    """calibration.py:113-122: fold one traced call (an object with `.activations`, or a dict
    name -> (IC, tokens) activations, numpy or CUDA) into the running mean of 2 X X^T, on the
    GPU in fp64."""
    import torch
    acts = trace.activations if hasattr(trace, "activations") else trace
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    contrib = {}
    for name, x in acts.items():
        xd = (x if hasattr(x, "is_cuda") else torch.from_numpy(np.ascontiguousarray(x))).to(
            dev, dtype=torch.float64)
        if xd.dim() != 2:
            raise ShapeError(f"layer {name}: activations must be (IC, tokens)")
        contrib[name] = torch.matmul(xd, xd.T).mul_(2.0)
    if running is None:
        return HessianFull(h=contrib, sample_count=1)
    if set(running.h) != set(contrib):
        raise ShapeError("trace layer set does not match running state")
    n = running.sample_count
    h = {}
    for name, c in contrib.items():
        prev = running.h[name]
        prev = prev if hasattr(prev, "is_cuda") else torch.from_numpy(np.asarray(prev, np.float64)).to(dev)
        if prev.shape != c.shape:
            raise ShapeError(f"layer {name}: IC {c.shape[0]} does not match running {prev.shape[0]}")
        h[name] = (prev * n + c) / (n + 1)
    return HessianFull(h=h, sample_count=n + 1)


@dataclass
class GlobalWeakColumns:
    k: int
    resid_indices: np.ndarray
    ffn_indices: list
    wo_indices: list
    s_global: np.ndarray


def accumulate_hessian_diag(activations: dict, running: HessianDiag | None = None) -> HessianDiag:
    """Fold one traced call (name -> (IC, tokens) activations) into the running
    mean (calibration.py:73-98). Accepts numpy arrays or CUDA tensors."""
    contrib = {}
    for name, x in activations.items():
        if hasattr(x, "is_cuda"):
            import torch
            contrib[name] = (2.0 * (x.double() ** 2).sum(dim=1)).cpu().numpy()
        else:
            contrib[name] = 2.0 * np.sum(np.asarray(x, np.float64) ** 2, axis=1)
    if running is None:
        return HessianDiag(lam=contrib, sample_count=1)
    if set(running.lam) != set(contrib):
        raise ShapeError("trace layer set does not match running state")
    n = running.sample_count
    lam = {}
    for name, c in contrib.items():
        prev = running.lam[name]
        if prev.shape != c.shape:
            raise ShapeError(f"layer {name}: IC {c.shape[0]} does not match running {prev.shape[0]}")
        lam[name] = (prev * n + c) / (n + 1)
    return HessianDiag(lam=lam, sample_count=n + 1)


def select_local_topk(scores, k: int) -> np.ndarray:
    """k largest scores, ties to the lower index, returned ascending."""
    scores = np.asarray(scores)
    if k > scores.shape[0]:
        raise ShapeError(f"k={k} exceeds {scores.shape[0]} channels")
    if k == 0:
        return np.zeros(0, dtype=np.int64)
    return np.sort(np.argsort(-scores, kind="stable")[:k]).astype(np.int64)


def select_global(hd: HessianDiag, k: int, *, n_blocks: int, layer_order=None) -> GlobalWeakColumns:
    """Pool mean-normalized lambda of every residual-fed layer at its local
    top-k into one residual-space set; per-block d_ff and wo sets stay local."""
    resid = [n for n in hd.lam if n == HEAD_NAME or n.split(".")[-1] in RESID_SUFFIXES]
    if layer_order is not None:
        resid = [n for n in layer_order if n in resid]
    if not resid:
        raise ShapeError("no residual-fed layers in the Hessian diagonal")
    d = hd.lam[resid[0]].shape[0]
    s = np.zeros(d, dtype=np.float64)
    for name in resid:
        lam = hd.lam[name].astype(np.float64)
        if lam.shape[0] != d:
            raise ShapeError(f"layer {name} IC {lam.shape[0]} != {d}")
        ids = select_local_topk(lam, k)
        mean = lam.mean()
        if mean > 0:
            s[ids] += lam[ids] / mean
    ffn, wo = [], []
    for i in range(n_blocks):
        ld, lw = hd.lam.get(f"b{i}.w_down"), hd.lam.get(f"b{i}.wo")
        if ld is None or lw is None:
            raise ShapeError(f"block {i} layers missing from Hessian diagonal")
        ffn.append(select_local_topk(ld, k))
        wo.append(select_local_topk(lw, k))
    return GlobalWeakColumns(k=k, resid_indices=select_local_topk(s, k), ffn_indices=ffn,
                             wo_indices=wo, s_global=s)
