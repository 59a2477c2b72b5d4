"""GPU quantizer kernels: alpha-grid parameter search and nearest codes,
bit-exact with the reference's grid_search_group_params / _nearest_codes
(pkg/src/qeft/quantizer.py:144-179, 211-218) -- same fp64 op order, numpy pairwise sums."""

import numpy as np
import pytest

from oracle import qeft_oracle as O
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import quantizer
    return quantizer


def _oracle_params(w, g, bits, steps, amin):
    oc, m = w.shape
    wd = w.astype(np.float32)
    return O.layer_params(wd, bits, g, "grid", steps, amin)


def test_grid_golden_segments(Q):
    """The reference's own grid results on fp32-valued segments (tests/golden/quantizer.npz)."""
    z = load_golden("quantizer")
    segs = z["grid_segs32"]
    sc, zr = Q._grid_params_gpu(segs, segs.shape[1], 4, 100, 0.5)
    assert np.array_equal(sc[:, 0], z["grid_scale32"]) and np.array_equal(zr[:, 0], z["grid_zero32"])
    sc, zr = Q._grid_params_gpu(np.ascontiguousarray(segs[:, :53]), 53, 3, 100, 0.5)
    assert np.array_equal(sc[:, 0], z["grid_scale32_b3_n53"])
    assert np.array_equal(zr[:, 0], z["grid_zero32_b3_n53"])


@pytest.mark.parametrize("oc,m,g,bits,steps,amin", [
    (48, 1000, 128, 4, 100, 0.5),   # ragged last group (104)
    (16, 700, 256, 4, 100, 0.5),    # groups > 128: numpy's recursive pairwise split
    (40, 333, 37, 3, 100, 0.5),     # odd group size, 3-bit
    (24, 200, 64, 4, 7, 0.8),       # few steps, other alpha_min
    (24, 200, 64, 3, 1, 0.5),       # steps = 1 is min-max
    (8, 5, 128, 4, 100, 0.5),       # a single group shorter than 8
])
def test_grid_params_bit_exact(Q, oc, m, g, bits, steps, amin):
    rng = np.random.default_rng(oc * 1000 + m)
    w = (rng.standard_normal((oc, m)) * 0.05).astype(np.float32)
    w[0, :] = 0.25                              # constant row -> (1, wmin)
    if m > 10:
        w[1, 3] = 4.0                           # an outlier group
        w[2, :: 3] = np.round(w[2, :: 3] * 8) / 8  # duplicated values: exact ties
    g_eff = min(g, m)
    sc, zr = Q._grid_params_gpu(w, g_eff, bits, steps, amin)
    so, zo = _oracle_params(w, g_eff, bits, steps, amin)
    assert np.array_equal(sc, so), np.argwhere(sc != so)[:5]
    assert np.array_equal(zr, zo), np.argwhere(zr != zo)[:5]
    codes = Q._nearest_codes_gpu(w, sc, zr, g_eff, bits)
    assert np.array_equal(codes, O.nearest_codes(w, so, zo, g_eff, bits))


def test_grid_cfg1_layer_bit_exact(Q):
    """A Cfg1-width slice (m = 3968, g = 128): every (row, group) equal to the oracle."""
    rng = np.random.default_rng(7)
    w = (rng.standard_normal((64, 3968)) * 0.02).astype(np.float32)
    sc, zr = Q._grid_params_gpu(w, 128, 4, 100, 0.5)
    so, zo = _oracle_params(w, 128, 4, 100, 0.5)
    assert np.array_equal(sc, so) and np.array_equal(zr, zo)


@pytest.mark.parametrize("oc,m,g,bits", [
    (96, 320, 64, 4),     # 5 blocks of 64 columns
    (130, 200, 48, 3),    # ragged groups and a partial last block, rows not a multiple of 64
    (64, 1000, 128, 4),   # 16 blocks, ragged last group
])
def test_optq_codes_bit_exact(Q, oc, m, g, bits, monkeypatch):
    """OPTQ codes equal the reference loop's given the reference's own factor (QEFT_OPTQ_FACTOR
    =host: same machine -> same LAPACK factor); with the GPU factor (cuSOLVER, the default) the
    codes agree to >= 99.9% (a factor entry one ulp away can move a value across a rounding
    boundary, and the error feedback carries it along the row)."""
    monkeypatch.setenv("QEFT_OPTQ_FACTOR", "host")
    rng = np.random.default_rng(oc + m)
    w = (rng.standard_normal((oc, m)) * 0.05).astype(np.float32)
    x = rng.standard_normal((m, 4 * m // 3))
    x[rng.choice(m, m // 16, replace=False)] *= 10.0
    h = 2.0 * x @ x.T
    sc, zr = Q._grid_params_gpu(w, g, bits, 100, 0.5)
    codes = Q._optq_gpu(w, h, sc, zr, g, bits)
    ref, fb = O.optq_codes(w, h, sc, zr, g, bits)
    assert not fb
    assert np.array_equal(codes, ref), (np.mean(codes == ref), np.argwhere(codes != ref)[:5])
    monkeypatch.setenv("QEFT_OPTQ_FACTOR", "device")
    dev = Q._optq_gpu(w, h, sc, zr, g, bits)
    assert np.mean(dev == ref) >= 0.999, np.mean(dev == ref)


def test_optq_fallback_on_singular_hessian(Q):
    """A non-positive-definite damped Hessian falls back to nearest rounding (quantizer.py:242-243)."""
    m = 64
    w = (np.random.default_rng(3).standard_normal((32, m)) * 0.05).astype(np.float32)
    h = -np.eye(m)
    sc, zr = Q._grid_params_gpu(w, 32, 4, 100, 0.5)
    assert Q._optq_gpu(w, h, sc, zr, 32, 4) is None          # device factor (cholesky fails)
    import torch
    assert Q._optq_factor_device(torch.from_numpy(h).cuda()) is None
    q = Q.quantize_layer(np.concatenate([w, w[:, :8]], 1), k=8, bits=4, g=32, mode="optq", h=-np.eye(72))
    assert q.optq_fallback
