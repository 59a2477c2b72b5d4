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
    """Y = W_hat_full @ X, saving only X[weak] (tuning.py:52-72). x: (IC, T) f32; the product
    runs in the tcgen05 forward GEMM (fp16 operands, fp32 accumulation)."""
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
    # the tcgen05 GEMM at every T: the same dequantized weights as the backward's dX GEMM, so
    # the gradients are those of this forward (the decode GEMV's fp16 (scale, zero) pairs serve
    # inference only: QuantLinearInferOp, KernelPathOp, the decode stack)
    y = dl.gemm_fwd(xt)
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
    """One optimizer step's work for `rank` of `world`: [(index, inputs, targets, weight)].

    Every rank draws the full stream of `grad_accum` micro-batches of `batch` windows from the
    shared generator, in the reference's order (tuning.py:209-213), so the generator stays in
    lockstep and the union over ranks is exactly the reference's accumulation group.
      world <= grad_accum: rank r takes whole micro-batches i with i % world == r (weight 1);
      world  > grad_accum: the grad_accum * batch windows are dealt round-robin (window w to
                           rank w % world) so no rank idles; a rank's windows are cut into
                           chunks of <= batch windows, each weighted n_windows / batch.
    The caller backpropagates weight * mean-loss(chunk) and divides the summed gradients by
    grad_accum, which reproduces the reference's sum-of-micro-batch-means / grad_accum
    (tuning.py:219-228) for every world size (exactly when the weights are powers of two).
    """
    draws = [sample_windows(rng, ids, cfg.batch, cfg.seq_len) for _ in range(cfg.grad_accum)]
    if world <= cfg.grad_accum:
        return [(i, xb, yb, 1.0) for i, (xb, yb) in enumerate(draws) if i % world == rank]
    xs = np.concatenate([d[0] for d in draws])
    ys = np.concatenate([d[1] for d in draws])
    mine = np.arange(rank, xs.shape[0], world)
    out = []
    for c in range(0, mine.size, cfg.batch):
        idx = mine[c:c + cfg.batch]
        out.append((c // cfg.batch, xs[idx], ys[idx], idx.size / cfg.batch))
    return out


def dp_allreduce_(grad, loss_sum, group=None):
    """Sum the flat weak-gradient bucket (None: already reduced bucket by bucket during the
    backward, WeakTrainer.arm_overlap) and the loss sum over the DP group; a no-op for a single
    process."""
    import torch.distributed as dist
    if group is not None and dist.get_world_size(group) > 1:
        if grad is not None:
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
        self.max_rows = max((l.oc for l in self.lins), default=0)
        self.step_no = 0
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.sq = torch.zeros(1, dtype=torch.float64, device=dev)
        # per-block buckets for the overlapped all-reduce: a contiguous slice of
        # the flat bucket per decoder block, launched as soon as the block's last dW lands
        blk = [l.name.split(".")[0] if "." in l.name else str(i) for i, l in enumerate(self.lins)]
        self.bucket_of, self.bucket_range, self.bucket_size = [], [], []
        for i, b in enumerate(blk):
            if not self.bucket_range or blk[i - 1] != b:
                self.bucket_range.append([int(self.offsets[i]), int(self.offsets[i + 1])])
                self.bucket_size.append(0)
            self.bucket_range[-1][1] = int(self.offsets[i + 1])
            self.bucket_size[-1] += 1
            self.bucket_of.append(len(self.bucket_range) - 1)
        self._pending = None
        self._works = []
        for i, l in enumerate(self.lins):
            l.grad_ready_hook = (lambda mod, i=i: self._grad_ready(i))

    def arm_overlap(self):
        """The next backward is the step's last on this rank: all-reduce every block's bucket
        on the collective's own stream as soon as all of its layers' dW_weak are in."""
        import torch.distributed as dist
        if self.group is None or dist.get_world_size(self.group) <= 1:
            return
        self._pending = list(self.bucket_size)

    def _grad_ready(self, i):
        if self._pending is None:
            return
        b = self.bucket_of[i]
        self._pending[b] -= 1
        if self._pending[b] == 0:
            self._launch(b)

    def _launch(self, b):
        import torch.distributed as dist
        lo, hi = self.bucket_range[b]
        self._works.append(dist.all_reduce(self.grad[lo:hi], group=self.group, async_op=True))
        self._pending[b] = -1

    def flush_overlap(self):
        """Launch the buckets that did not fire (layers without a weak block or no backward)."""
        if self._pending is None:
            return
        for b, c in enumerate(self._pending):
            if c >= 0:
                self._launch(b)

    def wait_allreduce(self):
        """Make the current stream wait for the launched bucket all-reduces."""
        if self._pending is not None:
            self.flush_overlap()
        for w in self._works:
            w.wait()
        self._works = []
        self._pending = None

    @property
    def n_params(self) -> int:
        return int(self.offsets[-1])

    def zero_grad(self):
        self.grad.zero_()

    def step(self, n_micro_total: int, loss_sum=None, reduced: bool = False):
        """All-reduce (DP, unless `reduced`) -> /(grad_accum * loss_scale) -> clip -> Adam
        -> weak16 refresh, in two passes over the bucket (libqeft_b200 qeft_grad_sqnorm_div +
        qeft_adam_step_flat; the divide is folded into both, the grads are left untouched).
        Returns the pre-clip global gradient norm squared (device fp64)."""
        import torch
        from . import optim
        cfg = self.cfg
        if not reduced:
            if loss_sum is None:
                loss_sum = torch.zeros((), dtype=torch.float64, device=self.grad.device)
            dp_allreduce_(self.grad, loss_sum, self.group)
        self.wait_allreduce()
        div = float(n_micro_total) * self.loss_scale  # loss_scale is a power of two: exact
        optim.grad_sqnorm_div(self.grad, div, out=self.sq)
        self.step_no += 1
        self.flag.zero_()
        optim.adam_step_flat(self.w32, self.m, self.v, self.grad, self.descs, len(self.lins), self.max_rows, div,
                             self.step_no, cfg.lr, max_norm=cfg.max_grad_norm, sqnorm=self.sq, flag=self.flag,
                             beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps)
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
        work = rank_micro_batches(rng, ids, cfg, rank, world)
        for ci, (_, xb, yb, wgt) in enumerate(work):
            if ci == len(work) - 1:
                tr.arm_overlap()  # the last backward all-reduces each block's bucket as it lands
            xt = torch.from_numpy(np.asarray(xb, np.int64)).to(dev)
            yt = torch.from_numpy(np.asarray(yb, np.int64)).to(dev)
            loss = cross_entropy_mean(model(xt), yt)
            (loss * (loss_scale * wgt)).backward()
            loss_sum += loss.detach().double() * wgt
        if not work:  # nothing to backprop on this rank: its (zero) bucket still joins the sum
            tr.arm_overlap()
            tr.flush_overlap()
        dp_allreduce_(None, loss_sum, group)
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
