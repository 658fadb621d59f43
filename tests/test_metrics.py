"""CPU: the evaluation metrics (reference metrics.py:98-241) score the same
seeded job batches to the same JSON documents as the reference's evaluate()
and aggregate() (goldens: tests/golden/make_golden_metrics.py), and
evaluate_sweep scores a batched replay's result records directly."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import golden
from metrics_cases import batches
from paper_2504_03887_b200 import metrics as M
from paper_2504_03887_b200.errors import EmptyInput, ZeroSize


def _jobs(raw):
    return [M.EvalJob(j["config_id"], j["predicted_peak"], j["capacity"],
                      j["oom_predicted"], M.ValidationRecord(**j["round1"]),
                      M.ValidationRecord(**j["round2"]) if j["round2"] else None)
            for j in raw]


@pytest.mark.parametrize("k", range(6))
def test_evaluate_matches_reference(k):
    raw = batches()[k]
    want = golden("metrics_golden.json")[k]
    got = M.evaluate(_jobs(raw))
    assert json.dumps(got, sort_keys=True) == json.dumps(want["evaluate"], sort_keys=True)
    agg = M.aggregate([(r["correctness_r1"], r["relative_error"] or 0.0)
                       for r in got["jobs"]]).to_json_dict()
    assert agg == want["aggregate"]


def test_scalar_helpers_and_errors():
    assert M.quadrant(0.1, 0.1) is M.Quadrant.OPTIMAL
    assert M.quadrant(0.3, 0.1) is M.Quadrant.UNDERESTIMATION
    assert M.quadrant(0.1, 0.3) is M.Quadrant.OVERESTIMATION
    assert M.quadrant(0.2, 0.2) is M.Quadrant.WORST
    assert M.memory_saved(10, 4, True, True, True) == 10
    assert M.memory_saved(10, 4, True, False, False) == 6
    assert M.memory_saved(10, 4, True, False, True) == -10
    assert M.memory_saved(10, 4, False, True, False) == -10
    with pytest.raises(ZeroSize):
        M.relative_error(5, 0)
    with pytest.raises(EmptyInput):
        M.evaluate([])
    with pytest.raises(EmptyInput):
        M.avg_memory_saved([])
    with pytest.raises(ValueError):
        M.ValidationRecord("a", 3, 0, "", 1, False)


def test_evaluate_sweep_from_result_records():
    from paper_2504_03887_b200._native import RESULT_DTYPE
    res = np.zeros(4, dtype=RESULT_DTYPE)
    res["peak_reserved"] = [10, 20, 30, 40]
    res["status"] = [0, 0, 1, 0]
    doc = M.evaluate_sweep(res, 25, actual_peak=[9, 21, 0, 50],
                           actual_oom=[False, False, True, True])
    jobs = [M.EvalJob(str(i), int(p), 25, o, M.ValidationRecord(str(i), 1, 0, "", a, ao))
            for i, (p, o, a, ao) in enumerate(zip([10, 20, 30, 40],
                                                   [False, False, True, True],
                                                   [9, 21, 0, 50],
                                                   [False, False, True, True]))]
    assert doc == M.evaluate(jobs)
