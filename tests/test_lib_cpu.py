"""CPU-side checks of the product package: the C-ABI library loads and exports
every symbol include/qeft_b200.h declares, the ctypes struct matches the C
layout, and the host-side format / index logic matches the oracle. No kernel
is launched here (no GPU in the build container)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import qeft_oracle as O
from tests.conftest import ROOT, load_golden


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "qeft_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(qeft_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2410_08661_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert b"sm_100a" in _lib.lib().qeft_version()


def test_struct_layout():
    from paper_2410_08661_b200 import _lib
    assert ctypes.sizeof(_lib.QeftLinearT) == 12 * 4 + 5 * 8
    assert _lib.QeftLinearT.qweight.offset == 48
    assert ctypes.sizeof(_lib.ShadowDescT) == 32


def test_qweight_bytes_formula():
    from paper_2410_08661_b200 import _lib
    L = _lib.lib()
    assert L.qeft_qweight_bytes(4096, 3968, 4) == 4096 * 3968 // 2
    assert L.qeft_qweight_bytes(17, 129, 3) == 2 * (256 * 6)


def test_host_pack_matches_oracle():
    from paper_2410_08661_b200 import packing
    z = load_golden("packing")
    for t in range(int(z["n"])):
        codes, bits = z[f"c{t}_codes"], int(z[f"c{t}_bits"])
        assert packing.pack_codes(codes, bits) == z[f"c{t}_packed"].tobytes()
        oc, m = codes.shape
        assert np.array_equal(packing.unpack_codes(z[f"c{t}_packed"].tobytes(), oc, m, bits), codes)


def test_selection_bit_exact():
    from paper_2410_08661_b200 import calibration, reorder
    z = load_golden("selection")
    for t in range(int(z["n"])):
        names = [str(s) for s in z[f"s{t}_names"]]
        hd = calibration.HessianDiag(lam={nm: z[f"s{t}_lam_{nm}"] for nm in names}, sample_count=1)
        gwc = calibration.select_global(hd, int(z[f"s{t}_k"]), n_blocks=2)
        assert np.array_equal(gwc.resid_indices, z[f"s{t}_resid"])
        assert np.array_equal(gwc.s_global, z[f"s{t}_sglobal"])
        for b in range(2):
            assert np.array_equal(gwc.ffn_indices[b], z[f"s{t}_ffn{b}"])
            assert np.array_equal(gwc.wo_indices[b], z[f"s{t}_wo{b}"])
        assert np.array_equal(reorder.weak_to_tail(24, gwc.resid_indices).perm, z[f"s{t}_perm"])
        run = None
        for x in z[f"s{t}_lx"]:
            run = calibration.accumulate_hessian_diag({"l": x}, run)
        assert np.array_equal(run.lam["l"], z[f"s{t}_lam_stream"])


def test_tile_code_addressing_is_a_bijection():
    """Every (row, col) of a 16 x m_pad block maps to a distinct bit field."""
    from paper_2410_08661_b200 import layer  # noqa: F401  (import check)
    for bits in (3, 4):
        m_pad = 256
        locs = [_locate(bits, m_pad, r, j) for r in range(16) for j in range(m_pad)]
        if bits == 4:
            assert len(set(locs)) == 16 * m_pad
        else:
            assert len({l[1] for l in locs}) == 16 * m_pad   # 2-bit fields
            assert len({l[2] for l in locs}) == 16 * m_pad   # hi bits


def _locate(bits, m_pad, r, j):
    # python mirror of qeft::locate_code (csrc/qeft_common.cuh) for the bijection test
    g, upper = r & 7, (r & 15) >> 3
    if bits == 4:
        kt, jc = j >> 6, j & 63
        t, sub, e = jc >> 4, (jc >> 2) & 3, jc & 3
        nib = (4 if e & 1 else 0) + (2 if e & 2 else 0) + upper
        return ("w", (kt * 128) + (4 * g + t) * 4 + sub, 4 * nib)
    kt, jc = j >> 7, j & 127
    h, jh = jc >> 6, jc & 63
    t, sub, e = jh >> 4, (jh >> 2) & 3, jh & 3
    ww, pp = sub >> 1, (e >> 1) * 2 + upper
    p, hs = 4 * (sub & 1) + pp, e & 1
    lo = (kt * 192 + (4 * g + t) * 4 + 2 * h + ww, 2 * p + 16 * hs)
    hi = (kt * 192 + 128 + (4 * g + t) * 2 + h, ((18 if hs else 2) + p + 8 * ww) & 31)
    return ("3", lo, hi)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2410_08661_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
