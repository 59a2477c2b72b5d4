"""Weak-column fine-tuning on B200 (reference API of pkg/src/qeft/tuning.py).

Same names and contracts as the reference:
  TrainableLayerState, CostCounters          tuning.py:30-49
  qlinear_forward_train / qlinear_backward   tuning.py:52-103
  QuantLinearTrainOp (engine linear-op)       tuning.py:106-131
  AdamState, adam_step                        tuning.py:137-160 (re-exported from optim)
  TuneConfig, finetune                        tuning.py:166-248
The numpy-facing functions keep the reference's (channels, tokens) orientation
and fp32 host arrays; the products run in the tcgen05 GEMMs of libqeft_b200.
Activations enter the kernels as fp16 scaled by an exact power of two (so the
fp16 grid is used at full precision whatever the caller's magnitude), and the
scale is divided back out of the fp32 results.

`finetune` runs the whole step on the GPU: a torch-hosted decoder
(model.QEFTDecoder) whose QEFTLinear layers write their weak-block gradients
into ONE flat fp32 bucket; with torch.distributed initialised, ranks take
disjoint micro-batches of the reference's window stream and the bucket is
all-reduced in a single NCCL call before the fused clip + Adam kernels.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import DivergenceError, ShapeError
from .layer import device_layer
from .optim import AdamState, adam_step  # noqa: F401  (reference names)


@dataclass
class TrainableLayerState:
    """tuning.py:30-34: the weak rows of the input, (k, T)."""
    x_weak: np.ndarray
    n_cols: int


@dataclass
class CostCounters:
    """tuning.py:37-49: exact weak-vs-full backward tallies."""
    wgrad_fma: int = 0
    full_fma: int = 0
    saved_elems: int = 0
    full_elems: int = 0

    def add(self, other: "CostCounters") -> None:
        self.wgrad_fma += other.wgrad_fma
        self.full_fma += other.full_fma
        self.saved_elems += other.saved_elems
        self.full_elems += other.full_elems


def _pow2_scale(a: np.ndarray) -> float:
    """Exact power of two bringing max|a| into [1, 2) (1.0 for all-zero input)."""
    m = float(np.max(np.abs(a))) if a.size else 0.0
    if not np.isfinite(m) or m == 0.0:
        return 1.0
    return float(2.0 ** (-math.floor(math.log2(m))))


def _to_dev(a: np.ndarray, scale: float):
    import torch
    return torch.from_numpy(np.ascontiguousarray((a * np.float32(scale)).T, np.float32)).cuda().half()


def qlinear_forward_train(q, x, *, w_hat_dense=None):
    """Y = W_hat_full @ X, saving only X[weak] (tuning.py:52-72). x: (IC, T) f32."""
    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[0] != q.ic:
        raise ShapeError(f"input rows {x.shape[0] if x.ndim else 0} != IC {q.ic}")
    T = x.shape[1]
    xs = x[q.input_perm] if q.input_perm is not None else x
    state = TrainableLayerState(x_weak=np.ascontiguousarray(xs[q.weak_indices]), n_cols=T)
    if T == 0:
        return np.zeros((q.oc, 0), np.float32), state
    dl = device_layer(q, "f16")
    s = _pow2_scale(x)
    xt = _to_dev(x, s)
    y = dl.gemm_fwd(xt) if T > 16 else dl.gemv(xt, out_f32=True)
    return (y.float().cpu().numpy().T / np.float32(s)).astype(np.float32), state


def dgrad_host(q, dy):
    """dX = W_hat_full^T @ dY (un-permuted for online layers) through the tcgen05 dgrad GEMM;
    dy (OC, T) f32 host -> (IC, T) f32 host. Also the frozen op's backward (qmodel.py:177-183)."""
    dy = np.asarray(dy, dtype=np.float32)
    t = dy.shape[1]
    if t == 0:
        return np.zeros((q.ic, 0), np.float32)
    dl = device_layer(q, "f16")
    sd = _pow2_scale(dy)
    dx = dl.gemm_dgrad(_to_dev(dy, sd)).float().cpu().numpy().T / np.float32(sd)
    return np.ascontiguousarray(dx, np.float32)


def qlinear_backward(state: TrainableLayerState, dy, q, *, w_hat_dense=None,
                     counters: CostCounters | None = None):
    """dX through the full W_hat, dW for the weak block only (tuning.py:75-103)."""
    import torch
    dy = np.asarray(dy, dtype=np.float32)
    t = state.n_cols
    if dy.shape != (q.oc, t):
        raise ShapeError(f"dY shape {dy.shape} != ({q.oc}, {t})")
    if counters is not None:
        counters.add(CostCounters(wgrad_fma=q.oc * q.k * t, full_fma=q.oc * q.ic * t,
                                  saved_elems=q.k * t, full_elems=q.ic * t))
    if t == 0:
        return np.zeros((q.ic, 0), np.float32), np.zeros((q.oc, q.k), np.float32)
    dl = device_layer(q, "f16")
    sd = _pow2_scale(dy)
    dyt = _to_dev(dy, sd)
    dx = dl.gemm_dgrad(dyt).float().cpu().numpy().T / np.float32(sd)
    dw = np.zeros((q.oc, q.k), np.float32)
    if q.k:
        sx = _pow2_scale(state.x_weak)
        kw = -(-q.k // 8) * 8
        xw = torch.zeros((t, kw), dtype=torch.float16, device="cuda")
        xw[:, :q.k] = _to_dev(state.x_weak, sx)
        dw = dl.gemm_wgrad_weak(dyt, xw).cpu().numpy() / np.float32(sd * sx)
    return np.ascontiguousarray(dx, np.float32), np.ascontiguousarray(dw, np.float32)


class QuantLinearTrainOp:
    """Engine linear-op protocol (model.py:192-216; tuning.py:106-131): plug into the
    reference engine via quant_engine(qm, op_factory=lambda nm, q: QuantLinearTrainOp(nm, q))."""

    always_weight_grad = True

    def __init__(self, name: str, q, counters: CostCounters | None = None):
        self.name = name
        self.q = q
        self.oc, self.ic = q.oc, q.ic
        self.counters = counters

    def apply(self, x2d):
        return qlinear_forward_train(self.q, x2d)[0]

    def forward_train(self, x2d):
        return qlinear_forward_train(self.q, x2d)

    def backward(self, state, dy2d, need_weight_grad=True):
        return qlinear_backward(state, dy2d, self.q, counters=self.counters)


# ---------------------------------------------------------------------------
# fine-tuning loop

@dataclass
class TuneConfig:
    """tuning.py:166-184 (same defaults)."""
    steps: int = 200
    lr: float = 5e-5
    batch: int = 4
    grad_accum: int = 4
    max_grad_norm: float = 0.3
    seq_len: int = 64
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0
    log_every: int = 25


def sample_windows(rng, ids, n, seq_len):
    """model.py:560-566: n random (seq_len+1)-token windows -> (inputs, targets)."""
    if len(ids) < seq_len + 1:
        raise ShapeError("corpus shorter than one training window")
    starts = rng.integers(0, len(ids) - seq_len - 1, size=n)
    w = np.stack([ids[s:s + seq_len + 1] for s in starts])
    return w[:, :-1], w[:, 1:]


def rank_micro_batches(rng, ids, cfg: TuneConfig, rank: int = 0, world: int = 1):
    """One optimizer step's micro-batches for `rank` of `world`.

    Every rank draws the full stream of `grad_accum` windows from the shared
    generator, in the reference's order (tuning.py:209-213), and keeps those with
    index % world == rank, so the union over ranks is exactly the reference's
    accumulation group and the generator stays in lockstep across ranks.
    Returns [(index, inputs, targets), ...].
    """
    out = []
    for i in range(cfg.grad_accum):
        xb, yb = sample_windows(rng, ids, cfg.batch, cfg.seq_len)
        if i % world == rank:
            out.append((i, xb, yb))
    return out


def dp_allreduce_(grad, loss_sum, group=None):
    """Sum the flat weak-gradient bucket and the loss sum over the DP group
    (one collective each; a no-op for a single process)."""
    import torch.distributed as dist
    if group is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, group=group)
        dist.all_reduce(loss_sum, group=group)
    return grad, loss_sum


class WeakTrainer:
    """Flat-bucket weak-column optimizer state for a QEFTDecoder.

    Every QEFTLinear's fp32 master and .grad become views into two flat fp32
    buffers (`w32`, `grad`), so one NCCL all-reduce covers all layers and clip +
    Adam is two fused launches (libqeft_b200 qeft_grad_sqnorm / qeft_adam_clip).
    """

    def __init__(self, model, cfg: TuneConfig, group=None, loss_scale: float = 1.0):
        import torch
        from . import optim
        self.model = model
        self.cfg = cfg
        self.group = group
        self.loss_scale = loss_scale
        self.lins = [l for l in model.linears() if l.k]
        sizes = [l.oc * l.k for l in self.lins]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        n = int(self.offsets[-1])
        dev = next(model.buffers()).device
        self.w32 = torch.empty(n, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(n, dtype=torch.float32, device=dev)
        self.m = torch.zeros(n, dtype=torch.float32, device=dev)
        self.v = torch.zeros(n, dtype=torch.float32, device=dev)
        for l, off, sz in zip(self.lins, self.offsets[:-1], sizes):
            self.w32[off:off + sz].copy_(l.weak32.data.reshape(-1))
            l.weak32.data = self.w32[off:off + sz].view(l.oc, l.k)
            l.weak32.grad = self.grad[off:off + sz].view(l.oc, l.k)
        self.descs, self.max_elems = optim.shadow_descs([l.dl for l in self.lins],
                                                        [int(o) for o in self.offsets[:-1]])
        self.step_no = 0
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.sq = torch.zeros(1, dtype=torch.float64, device=dev)

    @property
    def n_params(self) -> int:
        return int(self.offsets[-1])

    def zero_grad(self):
        self.grad.zero_()

    def step(self, n_micro_total: int, loss_sum=None, reduced: bool = False):
        """All-reduce (DP, unless `reduced`) -> /(grad_accum * loss_scale) -> clip -> Adam
        -> weak16 refresh. Returns the pre-clip global gradient norm (device fp64)."""
        import torch
        from . import optim
        cfg = self.cfg
        if not reduced:
            if loss_sum is None:
                loss_sum = torch.zeros((), dtype=torch.float64, device=self.grad.device)
            dp_allreduce_(self.grad, loss_sum, self.group)
        optim.div_(self.grad, float(n_micro_total) * self.loss_scale)
        optim.grad_sqnorm(self.grad, out=self.sq)
        self.step_no += 1
        self.flag.zero_()
        optim.adam_clip_(self.w32, self.m, self.v, self.grad, self.step_no, cfg.lr,
                         max_norm=cfg.max_grad_norm, beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps,
                         sqnorm=self.sq, flag=self.flag)
        optim.refresh_shadows(self.w32, self.descs, len(self.lins), self.max_elems)
        return self.sq


def _ddp_group():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.group.WORLD
    return None


def finetune(qm, dataset, config: TuneConfig | None = None, *, act_dtype: str = "f16",
             compute_dtype: str = "f32"):
    """Train the weak blocks of every quantized layer on next-token prediction
    (tuning.py:187-248). Returns (tuned QuantizedModel, log).

    Data parallel when torch.distributed is initialised: every rank draws the same
    window stream from `rng(seed)` (tuning.py:201, 213) and computes micro-batches
    i with i % world == rank, so the global step equals the reference's grad_accum
    micro-batches; the flat weak-gradient bucket is summed with one all-reduce.
    """
    import torch
    import torch.distributed as dist
    from .model import QEFTDecoder, cross_entropy_mean

    cfg = config or TuneConfig()
    tuned = qm.copy()
    if cfg.steps == 0:
        return tuned, []
    group = _ddp_group()
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    t_start = time.perf_counter()
    ids = np.asarray(dataset)
    rng = np.random.default_rng(cfg.seed)
    model = QEFTDecoder.from_quantized_model(tuned, act_dtype=act_dtype, compute_dtype=compute_dtype)
    # fp16 kernels: scale the loss so activation gradients sit well inside fp16 range;
    # the exact power of two is divided back out before clipping (reference grads in fp32)
    loss_scale = float(2 ** math.ceil(math.log2(cfg.batch * cfg.seq_len))) if act_dtype == "f16" else 1.0
    tr = WeakTrainer(model, cfg, group=group, loss_scale=loss_scale)
    per_micro = CostCounters()
    for l in tr.lins:
        t = cfg.batch * cfg.seq_len
        per_micro.add(CostCounters(wgrad_fma=l.oc * l.k * t, full_fma=l.oc * l.ic * t,
                                   saved_elems=l.k * t, full_elems=l.ic * t))
    log = []
    dev = tr.w32.device
    for step in range(1, cfg.steps + 1):
        tr.zero_grad()
        loss_sum = torch.zeros((), dtype=torch.float64, device=dev)
        for _, xb, yb in rank_micro_batches(rng, ids, cfg, rank, world):
            xt = torch.from_numpy(np.asarray(xb, np.int64)).to(dev)
            yt = torch.from_numpy(np.asarray(yb, np.int64)).to(dev)
            loss = cross_entropy_mean(model(xt), yt)
            (loss * loss_scale).backward()
            loss_sum += loss.detach().double()
        dp_allreduce_(tr.grad, loss_sum, group)
        loss_mean = float(loss_sum) / cfg.grad_accum
        if not math.isfinite(loss_mean):
            # the masters still hold the last finite update (tuning.py:215-218)
            raise DivergenceError(f"non-finite loss at step {step}", last_good=_export(tuned, tr),
                                  step=step)
        sq = tr.step(cfg.grad_accum, reduced=True)
        if int(tr.flag.item()):
            raise DivergenceError("non-finite gradient in adam_step", last_good=_export(tuned, tr),
                                  step=step)
        gnorm = math.sqrt(float(sq))
        if step % cfg.log_every == 0 or step == 1 or step == cfg.steps:
            log.append({"step": step, "loss": loss_mean, "grad_norm": gnorm,
                        "elapsed_s": round(time.perf_counter() - t_start, 3),
                        # cumulative, as the reference's counters (tuning.py:238-246)
                        "wgrad_fma": per_micro.wgrad_fma * cfg.grad_accum * step,
                        "full_fma": per_micro.full_fma * cfg.grad_accum * step,
                        "saved_elems": per_micro.saved_elems * cfg.grad_accum * step,
                        "full_elems": per_micro.full_elems * cfg.grad_accum * step})
    return _export(tuned, tr), log


def _export(tuned, tr: WeakTrainer):
    """Write the fp32 masters back into the host records (q.weak, in place)."""
    w = tr.w32.cpu().numpy()
    layers = dict(tuned.layer_items())
    for l, off in zip(tr.lins, tr.offsets[:-1]):
        layers[l.name].weak[...] = w[off:off + l.oc * l.k].reshape(l.oc, l.k)
    return tuned
