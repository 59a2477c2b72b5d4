"""Finite-difference gradient checks of the B200 train op -- the reference's criterion-4
harness (pkg/tests/test_tuning.py:93-137, pkg/tests/test_acceptance.py:150-197), re-run through
this package's qlinear_forward_train / qlinear_backward (tcgen05 GEMMs; the decode GEMV for
<= 16 tokens). Same tolerance: fd_relative_error <= 1e-2 (pkg/tests/conftest.py:158-161).

The kernels take fp16 operands, so a perturbation must survive the rounding to fp16 for a
central difference to mean anything: inputs and weak values are drawn on the 2^-6 grid with
|x| < 8, |w| < 2 (exactly representable in fp16). The forward is linear in both, so a central
difference is the exact derivative of the computed function at ANY step; the step is 16 (x +- 16
and w +- 16 stay exact in fp16), because the forward GEMM rounds y to fp16 (|y| ~ 10: ulp 2^-7)
and a one-grid-unit step would measure that rounding, not the gradient (measured: h = 1 leaves
up to 2 % FD noise, h = 16 below 1 %). dX uses the fp16 image of dY; dW_weak fp32 accumulation
of fp16 products. Training forwards always take the GEMM, so forward and backward share the
dequantized weights."""

import numpy as np
import pytest

from tests.conftest import fd_relative_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_08661_b200 import quantizer, tuning
    return quantizer, tuning


@pytest.mark.parametrize("t_range,g", [((2, 8), 8), ((17, 40), 8), ((2, 8), 64)])
def test_gradients_match_finite_differences(P, t_range, g):
    """20 random layer instances (reference: oc 4-24, ic 8-40, k 1-7, 4-bit, RTN, structured);
    short (T <= 16) and long token counts, g = 8 (generic dequant) and g = 64."""
    quantizer, tuning = P
    bad = []
    for trial in range(20):
        rng = np.random.default_rng(500 + trial)
        oc = int(rng.integers(4, 24))
        ic = int(rng.integers(8, 40)) if g == 8 else int(rng.integers(72, 200))
        k = int(rng.integers(1, min(8, ic - 1)))
        w = rng.standard_normal((oc, ic)).astype(np.float32)
        q = quantizer.quantize_layer(w, k=k, bits=4, g=g, mode="rtn", layout="structured")
        q.weak = np.clip(np.round(q.weak * 64) / 64, -1.98, 1.98).astype(np.float32)
        t = int(rng.integers(*t_range))
        x = np.clip(np.round(rng.standard_normal((ic, t)) * 64) / 64, -7.9, 7.9).astype(np.float32)
        dy = rng.standard_normal((oc, t)).astype(np.float32)
        _, state = tuning.qlinear_forward_train(q, x)
        dx, dw = tuning.qlinear_backward(state, dy, q)

        def loss():
            y, _ = tuning.qlinear_forward_train(q, x)
            return float(np.sum(y.astype(np.float64) * dy))

        wmax = max(float(np.abs(dw).max()), 1e-6)
        for _ in range(6):
            r, c = rng.integers(0, oc), rng.integers(0, k)
            orig = q.weak[r, c]
            h = 16.0
            q.weak[r, c] = orig + h
            lp = loss()
            q.weak[r, c] = orig - h
            lm = loss()
            q.weak[r, c] = orig
            e = fd_relative_error((lp - lm) / (2 * h), float(dw[r, c]), wmax)
            if e > 1e-2:
                bad.append(("w", trial, e))
        xmax = max(float(np.abs(dx).max()), 1e-6)
        for _ in range(6):
            r, c = rng.integers(0, ic), rng.integers(0, t)
            orig = x[r, c]
            h = 16.0
            x[r, c] = orig + h
            lp = loss()
            x[r, c] = orig - h
            lm = loss()
            x[r, c] = orig
            e = fd_relative_error((lp - lm) / (2 * h), float(dx[r, c]), xmax)
            if e > 1e-2:
                bad.append(("x", trial, e))
    assert not bad, bad[:10]
