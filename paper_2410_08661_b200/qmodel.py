"""Host containers of a quantized model (reference API names).

Mirrors pkg/src/qeft/qmodel.py:40-71 (QuantBlock, QuantizedModel) and the
architecture record of pkg/src/qeft/model.py:36-63 (ModelConfig), so records
built by the reference (or loaded from its fixtures) drop straight into
`finetune` and `QEFTDecoder.from_quantized_model`. Only the fields the hot path
reads are required; everything else is carried through untouched.
"""

from __future__ import annotations

import copy
from dataclasses import dataclass, field

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
    activation columns, the tcgen05 GEMM above. backward returns (dX, None): no weight grad."""

    def __init__(self, name: str, q):
        from .layer import device_layer
        self.name = name
        self.q = q
        self.oc, self.ic = q.oc, q.ic
        device_layer(q, "f16")  # build the device copy now (the reference's dequant-once)

    def apply(self, x2d):
        from .tuning import qlinear_forward_train
        return qlinear_forward_train(self.q, x2d)[0]

    def forward_train(self, x2d):
        return self.apply(x2d), None

    def backward(self, state, dy2d, need_weight_grad=True):
        from .tuning import dgrad_host
        return dgrad_host(self.q, dy2d), None
