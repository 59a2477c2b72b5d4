"""Host containers of a quantized model (reference API names).

Mirrors pkg/src/qeft/qmodel.py:40-71 (QuantBlock, QuantizedModel) and the
architecture record of pkg/src/qeft/model.py:36-63 (ModelConfig), so records
built by the reference (or loaded from its fixtures) drop straight into
`finetune` and `QEFTDecoder.from_quantized_model`. Only the fields the hot path
reads are required; everything else is carried through untouched.
"""

from __future__ import annotations

import copy
import hashlib
import json
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

BLOCK_LINEARS = ("wq", "wk", "wv", "wo", "w_up", "w_gate", "w_down")  # model.py:27
RESID_BLOCK_LINEARS = ("wq", "wk", "wv", "w_up", "w_gate")            # model.py:28
RMS_EPS = 1e-5                                                        # model.py:22
ROPE_BASE = 10000.0                                                   # model.py:23


@dataclass(frozen=True)
class ModelConfig:
    """model.py:36-63 (same defaults and validation)."""
    d_model: int = 64
    n_heads: int = 4
    head_dim: int = 16
    d_ff: int = 256
    n_blocks: int = 4
    vocab_size: int = 256
    max_seq: int = 128
    seed: int = 0

    def validate(self) -> None:
        for name in ("d_model", "n_heads", "head_dim", "d_ff", "n_blocks", "vocab_size", "max_seq"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.d_model != self.n_heads * self.head_dim:
            raise ConfigError(f"d_model ({self.d_model}) != n_heads ({self.n_heads}) * head_dim ({self.head_dim})")
        if self.d_ff < self.d_model:
            raise ConfigError(f"d_ff ({self.d_ff}) < d_model ({self.d_model})")
        if self.head_dim % 2 != 0:
            raise ConfigError("head_dim must be even (rotary pairs)")


# LLaMA-2 shapes (7B / 13B / 70B rows)
LLAMA2_7B = ModelConfig(d_model=4096, n_heads=32, head_dim=128, d_ff=11008, n_blocks=32,
                        vocab_size=32000, max_seq=2048)
LLAMA2_13B = ModelConfig(d_model=5120, n_heads=40, head_dim=128, d_ff=13824, n_blocks=40,
                         vocab_size=32000, max_seq=2048)


@dataclass
class DenseBlock:
    """model.py:66-80 BlockWeights: one decoder block's fp32 weights ((out, in) matrices)."""
    gain1: object
    wq: object
    wk: object
    wv: object
    wo: object
    gain2: object
    w_up: object
    w_gate: object
    w_down: object


@dataclass
class DenseModel:
    """model.py:83-99: the dense fp32 model quantize_model starts from (any object with these
    fields -- the reference's own DenseModel included -- is accepted)."""
    config: ModelConfig
    embedding: object
    blocks: list
    final_gain: object
    head: object

    def copy(self) -> "DenseModel":
        return copy.deepcopy(self)


REORDER_MODES = ("ogr", "online", "none")  # qmodel.py:38


def model_fingerprint(config) -> str:
    """qmodel.py:74-79: architecture hash; same-shape models match regardless of weights."""
    arch = {f: getattr(config, f) for f in
            ("d_model", "n_heads", "head_dim", "d_ff", "n_blocks", "vocab_size", "max_seq")}
    return hashlib.sha256(json.dumps(arch, sort_keys=True).encode()).hexdigest()[:16]


@dataclass
class QuantBlock:
    gain1: object
    gain2: object
    layers: dict  # wq/wk/wv/wo/w_up/w_gate/w_down -> QuantizedLinear


@dataclass
class QuantizedModel:
    """qmodel.py:47-71: frozen embedding / norms / dense head + quantized block linears."""
    config: ModelConfig
    embedding: object
    blocks: list
    final_gain: object
    head: object
    k: int = 0
    bits: int = 4
    g: int = 128
    mode: str = "rtn"
    reorder: str = "ogr"
    plan: object = None
    gwc: object = None
    fingerprint: str = ""
    meta: dict = field(default_factory=dict)

    def layer_items(self):
        """(name, QuantizedLinear) in canonical order (qmodel.py:64-67)."""
        for i, b in enumerate(self.blocks):
            for nm in BLOCK_LINEARS:
                yield f"b{i}.{nm}", b.layers[nm]

    def copy(self) -> "QuantizedModel":
        # device copies live in layer.DEVICE_CACHE, keyed by record: the copy gets its own
        return copy.deepcopy(self)


class QuantLinearInferOp:
    """Frozen quantized linear (qmodel.py:162-185), the reference's default op for
    quant_engine / quantized_perplexity (qmodel.py:206-224). The reference dequantizes once
    and multiplies dense fp32; here the layer is repacked once into the B200 layout
    (layer.device_layer) and every call runs the fused kernels: the decode GEMV for <= 16
    activation columns, the tcgen05 GEMM above. backward returns (dX, None): no weight grad.
    The kernel path reads x in the layer's input order; an online layer's colmap applies
    input_perm (as qlinear_forward_train does, tuning.py:64-65)."""

    def __init__(self, name: str, q):
        from .layer import device_layer
        self.name = name
        self.q = q
        self.oc, self.ic = q.oc, q.ic
        device_layer(q, "f16")  # build the device copy now (the reference's dequant-once)

    def apply(self, x2d):
        """<= 16 columns: the decode GEMV (one pass over the packed weights); more: the GEMM."""
        x2d = np.asarray(x2d, np.float32)
        if x2d.shape[1] <= 16:
            from .kernels import _run
            return _run(self.q, x2d, perm=None)
        from .tuning import qlinear_forward_train
        return qlinear_forward_train(self.q, x2d)[0]

    def forward_train(self, x2d):
        return self.apply(x2d), None

    def backward(self, state, dy2d, need_weight_grad=True):
        from .tuning import dgrad_host
        return dgrad_host(self.q, dy2d), None


def _np(a):
    return a.cpu().numpy() if hasattr(a, "is_cuda") else np.asarray(a)


def quantize_model(dense, hess, *, k: int = 8, bits: int = 4, g: int | None = 32, mode: str = "optq",
                   reorder: str = "ogr", grid_steps: int = 100, alpha_min: float = 0.5,
                   gwc=None, plan=None, meta: dict | None = None) -> QuantizedModel:
    """Quantize every block linear of a dense model (qmodel.py:82-156), on the GPU.

    `hess` is a calibration.HessianFull (per-layer 2 X X^T means in the ORIGINAL channel
    order; CUDA tensors from accumulate_hessian_full, or host arrays), reindexed to follow each
    layer's permutation. Reordering:
      ogr     select_global -> build_plan -> apply_ogr; every layer structured except wo,
              which stays irregular with its local weak set (qmodel.py:117-131);
      online  per-layer local top-k moved to the tail, input_perm stored (qmodel.py:132-141);
      none    per-layer local top-k, irregular layout (qmodel.py:142-147).
    Every quantize_layer call runs the GPU quantizer (RTN, or alpha-grid + OPTQ with the
    device fp64 factor). Passing gwc/plan reuses a previous selection."""
    from .calibration import select_global, select_local_topk
    from .errors import ConfigError
    from .quantizer import LAYOUT_IRREGULAR, LAYOUT_STRUCTURED, quantize_layer
    from .reorder import apply_ogr, build_plan, identity_plan, permute_hessian, weak_to_tail
    cfg = dense.config
    if reorder not in REORDER_MODES:
        raise ConfigError(f"reorder must be one of {REORDER_MODES}")
    lam = hess.diag()
    if reorder == "ogr":
        if gwc is None:
            gwc = select_global(lam, k, n_blocks=cfg.n_blocks)
        if plan is None:
            plan = build_plan(gwc, cfg)
        src = apply_ogr(dense, plan)
    else:
        gwc = None
        plan = identity_plan(cfg)
        src = dense.copy()
    blocks = []
    for i, b in enumerate(src.blocks):
        layers = {}
        for nm in BLOCK_LINEARS:
            name = f"b{i}.{nm}"
            w = _np(getattr(b, nm))
            h = hess.h[name]
            ge = g or w.shape[1] - k
            common = dict(k=k, bits=bits, g=ge, mode=mode, grid_steps=grid_steps, alpha_min=alpha_min)
            if reorder == "ogr":
                if nm == "wo":
                    layers[nm] = quantize_layer(w, layout=LAYOUT_IRREGULAR, indices=gwc.wo_indices[i], h=h,
                                                **common)
                else:
                    perm = plan.p_ffn[i] if nm == "w_down" else plan.p_resid
                    layers[nm] = quantize_layer(w, layout=LAYOUT_STRUCTURED, h=permute_hessian(h, perm),
                                                **common)
            elif reorder == "online":
                perm = weak_to_tail(w.shape[1], select_local_topk(lam.lam[name], k))
                q = quantize_layer(perm.apply_cols(w), layout=LAYOUT_STRUCTURED, h=permute_hessian(h, perm),
                                   **common)
                q.input_perm = perm.perm
                layers[nm] = q
            else:
                layers[nm] = quantize_layer(w, layout=LAYOUT_IRREGULAR,
                                            indices=select_local_topk(lam.lam[name], k), h=h, **common)
        blocks.append(QuantBlock(gain1=_np(b.gain1).copy(), gain2=_np(b.gain2).copy(), layers=layers))
    return QuantizedModel(config=cfg, embedding=_np(src.embedding).copy(), blocks=blocks,
                          final_gain=_np(src.final_gain).copy(), head=_np(src.head).copy(), plan=plan,
                          gwc=gwc, k=k, bits=bits, g=(g if g is not None else -1), mode=mode, reorder=reorder,
                          fingerprint=model_fingerprint(cfg), meta=dict(meta or {}))
