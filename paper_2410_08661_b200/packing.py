"""Reference-format code packing (host side) + the B200 tile conversion.

`row_bytes`, `pack_codes`, `unpack_codes` keep the reference's on-disk byte
format (pkg/src/qeft/packing.py:15-72: row-major, LSB-first, 4-bit even
column in the low nibble, 3-bit one bitstream per row padded to a byte) so
QuantizedLinear records interchange with the reference bit for bit. The
kernels never read this format: `to_tiles` / `from_tiles` convert on the GPU
to and from the B200 tile layout (csrc/qeft_common.cuh).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ShapeError


def row_bytes(m: int, bits: int) -> int:
    if bits == 4:
        return (m + 1) // 2
    if bits == 3:
        return (3 * m + 7) // 8
    raise ShapeError(f"unsupported bit width {bits}")


def pack_codes(codes, bits: int) -> bytes:
    """(OC, m) codes -> reference bytes (packing.py:24-52)."""
    codes = np.asarray(codes)
    if codes.ndim != 2:
        raise ShapeError(f"codes must be 2-D, got {codes.shape}")
    if bits not in (3, 4):
        raise ShapeError(f"unsupported bit width {bits}")
    if codes.size and (codes.min() < 0 or codes.max() >= (1 << bits)):
        raise ShapeError(f"code out of range for {bits}-bit packing")
    oc, m = codes.shape
    c = codes.astype(np.uint8)
    if bits == 4:
        if m % 2:
            c = np.pad(c, ((0, 0), (0, 1)))
        return (c[:, 0::2] | (c[:, 1::2] << 4)).tobytes()
    rb = row_bytes(m, 3)
    bitsarr = ((c[:, :, None] >> np.arange(3, dtype=np.uint8)) & 1).reshape(oc, 3 * m)
    bitsarr = np.pad(bitsarr, ((0, 0), (0, 8 * rb - 3 * m)))
    return np.packbits(bitsarr, axis=1, bitorder="little").tobytes()


def unpack_codes(data, oc: int, m: int, bits: int) -> np.ndarray:
    """Reference bytes -> (OC, m) uint8 codes (packing.py:55-72)."""
    rb = row_bytes(m, bits)
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    if raw.size != oc * rb:
        raise ShapeError(f"packed payload holds {raw.size} bytes, expected {oc * rb}")
    raw = raw.reshape(oc, rb)
    if bits == 4:
        out = np.stack([raw & 15, raw >> 4], axis=2).reshape(oc, 2 * rb)
        return np.ascontiguousarray(out[:, :m])
    b = np.unpackbits(raw, axis=1, bitorder="little")[:, :3 * m].reshape(oc, m, 3)
    return (b[:, :, 0] | (b[:, :, 1] << 1) | (b[:, :, 2] << 2)).astype(np.uint8)


def tile_bytes(oc: int, m: int, bits: int) -> int:
    return int(_lib.lib().qeft_qweight_bytes(oc, m, bits))


def to_tiles(packed, oc: int, m: int, bits: int, device="cuda"):
    """Reference bytes -> B200 tile layout (uint8 CUDA tensor), on the GPU."""
    import torch
    if bits not in (3, 4):
        raise ShapeError(f"unsupported bit width {bits}")
    ref = torch.from_numpy(np.frombuffer(bytes(packed), np.uint8).copy()).to(device)
    if ref.numel() != oc * row_bytes(m, bits):
        raise ShapeError("packed payload size mismatch")
    out = torch.empty(tile_bytes(oc, m, bits), dtype=torch.uint8, device=device)
    _lib.check(_lib.lib().qeft_repack_to_tiles(_lib.ptr(ref), oc, m, bits, _lib.ptr(out),
                                               _lib.stream_ptr()), "repack_to_tiles")
    return out


def from_tiles(qweight, oc: int, m: int, bits: int) -> bytes:
    """B200 tile layout -> reference bytes (bit-exact inverse of to_tiles)."""
    import torch
    out = torch.empty(oc * row_bytes(m, bits), dtype=torch.uint8, device=qweight.device)
    _lib.check(_lib.lib().qeft_repack_to_ref(_lib.ptr(qweight), oc, m, bits, _lib.ptr(out),
                                             _lib.stream_ptr()), "repack_to_ref")
    return out.cpu().numpy().tobytes()
