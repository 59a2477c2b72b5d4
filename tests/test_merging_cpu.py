"""Weak-delta merging against the reference's own outputs
(tests/golden/toy_*_tuned.qeft, toy_*.delta.qeft and container.npz, made by
tests/golden/make_golden.py container from pkg/src/qeft/merging.py)."""

import copy
import os

import numpy as np
import pytest

from paper_2410_08661_b200 import container as C
from paper_2410_08661_b200 import merging as Mg
from paper_2410_08661_b200.errors import MergeMismatchError
from tests.conftest import load_golden

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return C.load_checkpoint(os.path.join(GOLD, name))


@pytest.mark.parametrize("reo", ["ogr", "online"])
def test_extract_delta_matches_reference_file(reo):
    base, tuned = _load(f"toy_{reo}.qeft"), _load(f"toy_{reo}_tuned.qeft")
    ref_bytes = open(os.path.join(GOLD, f"toy_{reo}.delta.qeft"), "rb").read()
    d = Mg.extract_delta(tuned, base)
    assert C.dumps(d) == ref_bytes                      # same records, same bytes
    assert C.dumps(C.loads(ref_bytes)) == ref_bytes     # delta files re-save byte-identically
    assert d.plan_ref == Mg.plan_digest(base) == str(load_golden("container")[f"{reo}_plan_digest"])


@pytest.mark.parametrize("reo", ["ogr", "online"])
def test_apply_to_quantized_matches_reference(reo):
    z = load_golden("container")
    base = _load(f"toy_{reo}.qeft")
    merged = Mg.apply_to_quantized(base, C.loads(open(os.path.join(GOLD, f"toy_{reo}.delta.qeft"), "rb").read()))
    for name, q in merged.layer_items():
        assert np.array_equal(q.weak, z[f"{reo}_merged_{name}"]), name
    # the base is not modified
    assert C.dumps(base) == open(os.path.join(GOLD, f"toy_{reo}.qeft"), "rb").read()


def test_merge_mismatch_errors():
    base, tuned = _load("toy_ogr.qeft"), _load("toy_ogr_tuned.qeft")
    other = _load("toy_online.qeft")
    with pytest.raises(MergeMismatchError):      # frozen payloads differ
        Mg.extract_delta(other, base)
    d = Mg.extract_delta(tuned, base)
    with pytest.raises(MergeMismatchError):      # weak index sets differ
        Mg.apply_to_quantized(other, d)
    bad = copy.deepcopy(d)
    bad.fingerprint = "0" * 16
    with pytest.raises(MergeMismatchError):
        Mg.apply_to_quantized(base, bad)
