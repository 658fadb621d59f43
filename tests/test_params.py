"""Estimator parameter plumbing (reference base.py:8-40 via estimator.py:78):
get_params / set_params / repr behave like the reference's ParamMixin.  CPU
only; compared with the reference package itself when it is importable."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

from conftest import REPO
from paper_2504_03887_b200.estimator import PeakMemoryEstimator


def _reference():
    for cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if cand.exists() and str(cand) not in sys.path:
            sys.path.insert(0, str(cand))
    return pytest.importorskip("peakmem.estimator").PeakMemoryEstimator


def test_params_round_trip():
    est = PeakMemoryEstimator(iterations=3, max_split_size=1 << 20)
    params = est.get_params()
    assert list(params) == sorted(params)
    assert params["iterations"] == 3 and params["max_split_size"] == 1 << 20
    assert est.set_params(device_capacity=1 << 30) is est
    assert est.get_params()["device_capacity"] == 1 << 30
    assert repr(est).startswith("PeakMemoryEstimator(device_capacity=1073741824, ")


def test_unknown_parameter_after_known_ones():
    est = PeakMemoryEstimator()
    with pytest.raises(ValueError, match="invalid parameter 'bogus'"):
        est.set_params(iterations=5, bogus=1)
    assert est.iterations == 5  # set before the unknown name, as in the reference


def test_matches_reference():
    Ref = _reference()
    for kw in ({}, {"iterations": 4, "device_capacity": 1 << 34, "validate": True}):
        ours, ref = PeakMemoryEstimator(**kw), Ref(**kw)
        assert ours.get_params() == ref.get_params()
        assert repr(ours) == repr(ref)
    msgs = []
    for C in (PeakMemoryEstimator, Ref):
        with pytest.raises(ValueError) as err:
            C().set_params(bogus=1)
        msgs.append(str(err.value))
    assert msgs[0] == msgs[1]
