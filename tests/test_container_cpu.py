"""`.qeft` container against files written by the reference's own
save_checkpoint (tests/golden/toy_*.qeft, made by tests/golden/make_golden.py container):
byte-identical re-save, field parity with the independent finetune fixture, and the
reference's error behaviour (pkg/src/qeft/container.py:111-142; pkg/tests/test_container.py)."""

import os
import struct
import zlib

import numpy as np
import pytest

from paper_2410_08661_b200 import container as C
from paper_2410_08661_b200.errors import (BadMagicError, ChecksumError, ContainerError, TruncatedFileError,
                                          UnsupportedVersionError)
from paper_2410_08661_b200.qmodel import BLOCK_LINEARS
from tests.conftest import load_golden

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _data(reo):
    with open(os.path.join(GOLD, f"toy_{reo}.qeft"), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("reo", ["ogr", "online"])
def test_reference_file_resaves_byte_identically(reo, tmp_path):
    data = _data(reo)
    qm = C.loads(data)
    assert C.encode_quantized(qm) == data
    p = tmp_path / "m.qeft"
    C.save_checkpoint(p, qm)
    assert p.read_bytes() == data
    assert C.encode_quantized(C.load_checkpoint(p)) == data


@pytest.mark.parametrize("mi,reo", [(0, "ogr"), (1, "online")])
def test_loaded_fields_match_reference_model(mi, reo):
    """The same toy models (same seeds) as the finetune fixture, recorded field by field."""
    z = load_golden("finetune")
    qm = C.loads(_data(reo))
    pre = f"m{mi}_"
    assert np.array_equal(qm.embedding, z[pre + "embedding"]) and np.array_equal(qm.head, z[pre + "head"])
    assert np.array_equal(qm.final_gain, z[pre + "final_gain"])
    for i, b in enumerate(qm.blocks):
        assert np.array_equal(b.gain1, z[pre + f"b{i}_gain1"]) and np.array_equal(b.gain2, z[pre + f"b{i}_gain2"])
        for nm in BLOCK_LINEARS:
            q, p = b.layers[nm], pre + f"b{i}.{nm}_"
            assert q.packed == z[p + "packed"].tobytes()
            for f in ("scales", "zeros", "weak", "weak_indices"):
                assert np.array_equal(getattr(q, f), z[p + f]), (nm, f)
            perm = z[p + "input_perm"]
            assert (q.input_perm is None) == (perm.size == 0)
            if q.input_perm is not None:
                assert np.array_equal(q.input_perm, perm)
    assert qm.reorder == reo and (qm.gwc is not None) == (reo == "ogr")


def _reseal(body: bytes) -> bytes:
    return body + struct.pack("<I", zlib.crc32(body))


def test_container_errors():
    data = _data("ogr")
    with pytest.raises(BadMagicError):
        C.loads(b"QEFX" + data[4:])
    with pytest.raises(BadMagicError):
        C.loads(b"QE")
    with pytest.raises(TruncatedFileError):
        C.loads(data[:12])
    with pytest.raises(TruncatedFileError):
        C.loads(data[:len(data) // 2])
    with pytest.raises(ChecksumError):
        C.loads(data[:-4] + struct.pack("<I", zlib.crc32(data[:-4]) ^ 1))
    flipped = bytearray(data)
    flipped[len(data) // 3] ^= 0xFF
    with pytest.raises((ChecksumError, TruncatedFileError, UnicodeDecodeError)):
        C.loads(bytes(flipped))
    body = bytearray(data[:-4])
    struct.pack_into("<H", body, 4, 2)
    with pytest.raises(UnsupportedVersionError):
        C.loads(_reseal(bytes(body)))
    with pytest.raises(TruncatedFileError):  # trailing bytes after the last record
        C.loads(_reseal(data[:-4] + b"\x00"))
    body = bytearray(data[:-4])
    body[6] = C.KIND_DENSE
    with pytest.raises(ContainerError):
        C.loads(_reseal(bytes(body)))
    body[6] = 9
    with pytest.raises(UnsupportedVersionError):
        C.loads(_reseal(bytes(body)))
