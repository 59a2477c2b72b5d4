"""Pin the CPU oracle to the reference: golden vectors made by the reference
itself (tests/golden/make_golden.py) plus the reference tests' known answers.

CPU only (no gpu marker).
"""

import numpy as np
import pytest

from oracle import qeft_oracle as O
from tests.conftest import golden_layer, load_golden, rel_err


# --- packing: pkg/tests/test_packing.py:12-35 known answers -----------------

def test_pack_known_answers():
    assert O.pack_codes(np.array([[1, 2]]), 4) == b"\x21"
    assert O.pack_codes(np.array([[0xF, 0x3, 0x7]]), 4) == bytes([0x3F, 0x07])
    d = O.pack_codes(np.array([[1, 2, 3]]), 3)
    assert len(d) == O.row_bytes(3, 3) == 2 and d[0] == 0b11010001 and d[1] == 0
    assert O.pack_codes(np.zeros((3, 5), np.uint8), 4) == bytes(9)
    assert O.pack_codes(np.zeros((3, 5), np.uint8), 3) == bytes(6)
    data = O.pack_codes(np.array([[7, 7, 7], [1, 0, 1]], np.uint8), 3)
    assert O.unpack_codes(data, 2, 3, 3)[1].tolist() == [1, 0, 1]


@pytest.mark.parametrize("bad,bits", [([[16]], 4), ([[8]], 3), ([[-1]], 4), ([[1]], 5)])
def test_pack_errors(bad, bits):
    with pytest.raises(O.OracleShapeError):
        O.pack_codes(np.array(bad), bits)


def test_pack_golden_bit_exact():
    z = load_golden("packing")
    for t in range(int(z["n"])):
        codes, bits = z[f"c{t}_codes"], int(z[f"c{t}_bits"])
        packed = z[f"c{t}_packed"].tobytes()
        assert O.pack_codes(codes, bits) == packed
        oc, m = codes.shape
        assert np.array_equal(O.unpack_codes(packed, oc, m, bits), codes)


# --- quantizer: quantize_layer bit-exact vs reference -------------------------

def test_quantize_layer_golden_bit_exact():
    z = load_golden("quantizer")
    for n in range(int(z["n"])):
        p = f"q{n}_"
        mode = str(z[p + "mode"])
        kw = dict(k=int(z[p + "k"]), bits=int(z[p + "bits"]),
                  g=int(z[p + "g"]) if mode == "rtn" else None, mode=mode,
                  layout=str(z[p + "layout"]))
        ref = golden_layer(z, p)
        if mode == "optq":
            # the reference was called with the requested g; the stored g is g_eff
            kw["g"] = ref.g
            kw["x"] = z[p + "xcal"]
            if p + "lam" in z:
                kw["lam"] = z[p + "lam"]
        q = O.quantize_layer(z[p + "w"], **kw)
        assert q.g == ref.g
        assert q.packed == ref.packed, n
        assert np.array_equal(q.scales, ref.scales), n
        assert np.array_equal(q.zeros, ref.zeros), n
        assert np.array_equal(q.weak, ref.weak)
        assert np.array_equal(q.weak_indices, ref.weak_indices)
        assert bool(q.optq_fallback) == bool(z[p + "fallback"])


def test_grid_search_golden():
    z = load_golden("quantizer")
    s, zz = O.grid_scale_zero(np.array([0.0, 1.0, 2.0, 100.0]), 2)
    assert (s, zz) == tuple(z["grid_outlier_params"])
    for i, seg in enumerate(z["grid_segs"]):
        s, zz = O.grid_scale_zero(seg, 4)
        assert s == z["grid_scale"][i] and zz == z["grid_zero"][i]
    # fp32-valued segments (the quantize_layer input type), 4-bit and 3-bit over 53 values
    for i, seg in enumerate(z["grid_segs32"]):
        s, zz = O.grid_scale_zero(seg, 4)
        assert np.float32(s) == z["grid_scale32"][i] and np.float32(zz) == z["grid_zero32"][i]
        s, zz = O.grid_scale_zero(seg[:53], 3)
        assert np.float32(s) == z["grid_scale32_b3_n53"][i] and np.float32(zz) == z["grid_zero32_b3_n53"][i]
    # grid_steps=1 is min-max (pkg/tests/test_quantizer.py:59-63)
    seg = z["grid_segs"][0]
    assert O.grid_scale_zero(seg, 4, steps=1) == O.minmax_scale_zero(seg, 4)


def test_rtn_known_answers():
    # pkg/tests/test_quantizer.py:23-32: exact ramp, constant group
    s, zz = O.minmax_scale_zero(np.arange(16, dtype=np.float32), 4)
    assert (s, zz) == (1.0, 0.0)
    assert O.minmax_scale_zero(np.full(5, 2.5, np.float32), 4) == (1.0, 2.5)


def test_quantize_layer_structure():
    # pkg/tests/test_quantizer.py:170-210: k=0, weak passthrough, ragged, g>m
    rng = np.random.default_rng(0)
    w = rng.standard_normal((6, 15)).astype(np.float32)
    q = O.quantize_layer(w, k=4, bits=4, g=4, mode="rtn")
    assert q.m == 11 and q.n_groups == 3 and np.array_equal(q.weak, w[:, 11:])
    q0 = O.quantize_layer(w, k=0, bits=3, g=64, mode="rtn")
    assert q0.g == 15 and q0.n_groups == 1 and q0.weak.shape == (6, 0)
    with pytest.raises(O.OracleShapeError):
        O.quantize_layer(w, k=15, bits=4, g=4, mode="rtn")
    with pytest.raises(O.OracleShapeError):
        O.quantize_layer(w, k=2, bits=4, g=4, mode="rtn", indices=np.array([0, 1]))


# --- matvec -------------------------------------------------------------------

def test_matvec_golden():
    z = load_golden("quantizer")
    for n in range(int(z["n"])):
        p = f"q{n}_"
        q = golden_layer(z, p)
        x = z[p + "x"]
        assert rel_err(O.matvec_reference(q, x), z[p + "y_ref"]) == 0.0
        if p + "y_struct" in z:
            assert np.array_equal(O.matvec_structured(q, x), z[p + "y_struct"]), n
        if p + "y_irr" in z:
            assert np.array_equal(O.matvec_irregular(q, x), z[p + "y_irr"]), n


def test_matvec_counters_hand_computation():
    # pkg/tests/test_kernels.py:116-126
    q = O.quantize_layer(np.ones((8, 20), np.float32), k=4, bits=4, g=8, mode="rtn")
    m, ng, oc, k = 16, 2, 8, 4
    assert O.analytic_bytes(q) == oc * O.row_bytes(m, 4) + 2 * 4 * oc * ng + 4 * oc * k
    assert O.analytic_fmas(q) == oc * m + 2 * oc * ng + oc * k


def test_online_equals_structured_of_permuted():
    # pkg/tests/test_kernels.py:94-100 (bitwise)
    rng = np.random.default_rng(5)
    w = rng.standard_normal((8, 16)).astype(np.float32)
    q = O.quantize_layer(w, k=3, bits=4, g=5, mode="rtn")
    perm = rng.permutation(16)
    x = rng.standard_normal(16).astype(np.float32)
    assert np.array_equal(O.matvec_online_reorder(q, x, perm), O.matvec_structured(q, x[perm]))


# --- training fwd/bwd and Adam ------------------------------------------------

def test_train_fwd_bwd_golden():
    z = load_golden("training")
    for t in range(int(z["n"])):
        p = f"t{t}_"
        q = golden_layer(z, p)
        ip = z[p + "input_perm"]
        q.input_perm = ip if ip.size else None
        y, xw = O.forward_train(q, z[p + "x"])
        assert np.array_equal(y, z[p + "y"]) and np.array_equal(xw, z[p + "xw"])
        dx, dw = O.backward(q, xw, z[p + "dy"])
        assert np.array_equal(dx, z[p + "dx"]) and np.array_equal(dw, z[p + "dw"])
        c = O.cost_counters(q, xw.shape[1])
        assert [c["wgrad_fma"], c["full_fma"], c["saved_elems"], c["full_elems"]] == \
            z[p + "counters"].tolist()


def test_adam_golden():
    z = load_golden("training")
    for t in range(3):
        w = z[f"adam{t}_w0"].copy()
        st = O.AdamMoments(np.zeros_like(w), np.zeros_like(w))
        for s in range(6):
            O.adam_update(st, w, z[f"adam{t}_g"][s], lr=0.01 * (t + 1))
        assert np.array_equal(w, z[f"adam{t}_w"])
        assert np.array_equal(st.m, z[f"adam{t}_m"]) and np.array_equal(st.v, z[f"adam{t}_v"])


def test_adam_first_step_closed_form():
    # pkg/tests/test_tuning.py:146-155
    w = np.zeros((2, 2), np.float32)
    g = np.array([[1.0, -2.0], [0.5, 0.0]], np.float32)
    O.adam_update(O.AdamMoments(np.zeros_like(w), np.zeros_like(w)), w, g, lr=0.01)
    want = -0.01 * g / (np.abs(g) + 1e-8)
    assert np.allclose(w, want, rtol=1e-5)


# --- selection / reorder --------------------------------------------------------

def test_selection_golden():
    z = load_golden("selection")
    for t in range(int(z["n"])):
        names = [str(s) for s in z[f"s{t}_names"]]
        lam = {nm: z[f"s{t}_lam_{nm}"] for nm in names}
        resid, ffn, wo, s = O.select_global(lam, int(z[f"s{t}_k"]), n_blocks=2)
        assert np.array_equal(resid, z[f"s{t}_resid"])
        assert np.array_equal(s, z[f"s{t}_sglobal"])
        for b in range(2):
            assert np.array_equal(ffn[b], z[f"s{t}_ffn{b}"])
            assert np.array_equal(wo[b], z[f"s{t}_wo{b}"])
        assert np.array_equal(O.weak_to_tail(24, resid), z[f"s{t}_perm"])
        run, n = None, 0
        for x in z[f"s{t}_lx"]:
            run, n = O.lambda_running(run, n, x)
        assert np.array_equal(run, z[f"s{t}_lam_stream"])


def test_selection_known_answers():
    # pkg/tests/test_calibration.py:97-105 and test_reorder.py:38-53
    assert O.topk_ascending(np.array([0.8, 2.0]), 1).tolist() == [1]
    assert O.topk_ascending(np.array([5.0, 5.0, 1.0]), 1).tolist() == [0]
    assert O.weak_to_tail(4, [1]).tolist() == [0, 2, 3, 1]
    assert O.weak_to_tail(6, [1, 4]).tolist() == [0, 2, 3, 5, 1, 4]
    # select_global worked example (test_calibration.py:128-142): 1.6 vs 1.5 -> {0}
    lam = {"b0.wq": np.array([8.0, 2.0]), "b0.wk": np.array([1.0, 3.0]),
           "b0.wo": np.ones(2), "b0.w_down": np.ones(4)}
    resid, _, _, s = O.select_global(lam, 1, n_blocks=1)
    assert resid.tolist() == [0] and np.allclose(s, [1.6, 1.5])
