"""Shared test plumbing: the `gpu` marker, oracle import path, golden loader."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def golden_layer(z, prefix):
    """Rebuild an oracle layer record from a golden fixture entry."""
    from oracle.qeft_oracle import OracleLayer
    return OracleLayer(
        oc=int(z[prefix + "oc"]), ic=int(z[prefix + "ic"]), k=int(z[prefix + "k"]),
        bits=int(z[prefix + "bits"]), g=int(z[prefix + "g"]),
        packed=z[prefix + "packed"].tobytes(), scales=z[prefix + "scales"],
        zeros=z[prefix + "zeros"], weak=z[prefix + "weak"],
        weak_indices=z[prefix + "weak_indices"], layout=str(z[prefix + "layout"]))


def rel_err(y, ref):
    """The reference's metric: max|y-ref| / max(1, max|ref|) (pkg/tests/test_kernels.py:37)."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(y - ref)) / max(1.0, float(np.max(np.abs(ref)))))


def fd_relative_error(fd, an, scale):
    """pkg/tests/conftest.py:158-161: FD tolerance with a 2%-of-scale floor."""
    return abs(fd - an) / max(abs(fd), abs(an), 0.02 * scale)


@pytest.fixture(scope="session")
def golden():
    return load_golden
