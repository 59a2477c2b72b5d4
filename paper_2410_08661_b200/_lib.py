"""ctypes binding of libqeft_b200.so (include/qeft_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (nvcc,
sm_100a). There is no fallback: if the library or a GPU is missing, every
compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QEFT_LIB_PATH") or os.path.join(_HERE, "libqeft_b200.so")  # override: A/B tuning
CSRC = os.path.join(_HERE, "csrc")

QEFT_F16 = 0
QEFT_BF16 = 1
QEFT_FLAG_STRUCTURED_FAST = 1


class QeftLinearT(ctypes.Structure):
    """Mirror of qeft_linear_t (include/qeft_b200.h)."""
    _fields_ = [(n, ctypes.c_int32) for n in (
        "oc", "ic", "k", "bits", "g", "m", "ng", "m_pad", "k_pad", "oc_pad", "act_dtype", "flags")] + [
        ("qweight", ctypes.c_void_p), ("sz", ctypes.c_void_p), ("weak16", ctypes.c_void_p),
        ("colmap", ctypes.c_void_p), ("sz16", ctypes.c_void_p)]


class ShadowDescT(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("oc", ctypes.c_int32), ("k", ctypes.c_int32),
                ("k_pad", ctypes.c_int32), ("act_dtype", ctypes.c_int32), ("weak16", ctypes.c_void_p)]


# name -> (restype, argtypes); exactly the symbols include/qeft_b200.h declares
_VP, _I, _I64, _SZ, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float
_LP = ctypes.POINTER(QeftLinearT)
SIGNATURES = {
    "qeft_qweight_bytes": (_SZ, [_I, _I, _I]),
    "qeft_repack_to_tiles": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "qeft_repack_to_ref": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "qeft_pack_sz": (_I, [_VP, _VP, _I, _I, _VP, _VP]),
    "qeft_sz16_bytes": (_SZ, [_I, _I, _I]),
    "qeft_pack_sz16": (_I, [_VP, _VP, _I, _I, _I, _VP, _VP]),
    "qeft_pack_weak": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "qeft_dequant_full": (_I, [_LP, _VP, _VP]),
    "qeft_gather_cols": (_I, [_VP, _I64, _VP, _I, _I, _I, _VP, _VP]),
    "qeft_quantize_rtn": (_I, [_VP, _I, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "qeft_grid_params": (_I, [_VP, _I, _I, _I, _I, _I, ctypes.c_double, _VP, _VP, _VP]),
    "qeft_nearest_codes": (_I, [_VP, _I, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "qeft_optq_codes": (_I, [_VP, _VP, _VP, _VP, _I, _I, _I, _I, _VP, _VP, _VP]),
    "qeft_gemv_trace": (_I, [_I, _VP]),
    "qeft_gemm_set_schedule": (_I, [_I, _I]),
    "qeft_gemm_wgrad_weak_multi": (_I, [_VP, _I, _VP, _VP, _VP, _I64, _VP, _I, _I, _VP]),
    "qeft_gemv_multi_rmsnorm": (_I, [_VP, _I, _VP, _I64, _VP, _VP, _I64, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemv_swiglu": (_I, [_LP, _VP, _VP, _I64, _VP, _I64, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemv_workspace_bytes": (_SZ, [_LP, _I]),
    "qeft_gemv": (_I, [_LP, _VP, _I64, _VP, _I64, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemv_multi": (_I, [_VP, _I, _VP, _I64, _VP, _I64, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemm_workspace_bytes": (_SZ, [_LP, _I]),
    "qeft_gemm_fwd": (_I, [_LP, _VP, _I64, _VP, _I64, _I, _VP, _SZ, _VP]),
    "qeft_gemm_dgrad": (_I, [_LP, _VP, _I64, _VP, _I64, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemm_wgrad": (_I, [_LP, _VP, _I64, _VP, _I64, _VP, _I, _I, _VP, _SZ, _VP]),
    "qeft_gemm_wgrad_weak": (_I, [_LP, _VP, _I64, _VP, _I64, _VP, _I, _I, _VP, _SZ, _VP]),
    "qeft_grad_sqnorm": (_I, [_VP, _I64, _VP, _VP, _VP]),
    "qeft_div_scalar": (_I, [_VP, _I64, _F, _VP]),
    "qeft_adam_clip": (_I, [_VP, _VP, _VP, _VP, _I64, _VP, ctypes.c_double, _F, _F, _F, _F, _F, _F, _F, _F, _VP,
                            _VP]),
    "qeft_grad_sqnorm_div": (_I, [_VP, _I64, _F, _VP, _VP, _VP]),
    "qeft_adam_step_flat": (_I, [_VP, _VP, _VP, _VP, _VP, _I, _I, _F, _VP, ctypes.c_double, _F, _F, _F, _F, _F,
                                 _F, _F, _F, _VP, _VP]),
    "qeft_weak_shadow": (_I, [_VP, _VP, _I, _I, _VP]),
    "qeft_rmsnorm_fwd": (_I, [_VP, _VP, _VP, _VP, _I, _I, _I, _VP]),
    "qeft_rmsnorm_bwd": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _VP]),
    "qeft_rope": (_I, [_VP, _VP, _VP, _VP, _I64, _I, _I, _I, _I, _I, _VP]),
    "qeft_rope_kv": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I, _I, _VP]),
    "qeft_silu_mul_fwd": (_I, [_VP, _VP, _VP, _I64, _I, _VP]),
    "qeft_decode_attention": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I, _I, _VP, _SZ, _VP]),
    "qeft_decode_attention_workspace_bytes": (_SZ, [_I, _I, _I]),
    "qeft_cross_entropy_fwd": (_I, [_VP, _I64, _I, _I, _VP, _VP, _VP, _I, _VP]),
    "qeft_cross_entropy_bwd": (_I, [_VP, _I64, _I, _I, _VP, _VP, _VP, _VP, _I64, _I, _VP]),
    "qeft_silu_mul_bwd": (_I, [_VP, _VP, _VP, _VP, _VP, _I64, _I, _VP]),
    "qeft_last_error": (ctypes.c_char_p, []),
    "qeft_version": (ctypes.c_char_p, []),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree (make in csrc/)."""
    out = subprocess.run(["make", "-C", CSRC, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libqeft_b200 build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if verbose:
        print(out.stdout[-2000:])
    return LIB_PATH


def lib():
    """Load the library (once). Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


CALLS = [0]  # C-ABI calls made through check() (bench.py reports them per timed region)


def check(rc: int, what: str) -> None:
    CALLS[0] += 1
    if rc == 0:
        return
    msg = lib().qeft_last_error().decode(errors="replace")
    if rc in (1, 2):
        raise ShapeError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(t, what="tensor"):
    if not t.is_cuda:
        raise RuntimeError(f"{what} must be a CUDA tensor: the B200 path has no CPU fallback")
