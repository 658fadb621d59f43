"""Metrics: the OOM verdict on the estimation path (metrics.py:91-95) and the
paper's evaluation of many predictions against measured runs
(metrics.py:98-241, SURVEY §8f f3 "evaluate() at scale").

Evaluation is column-oriented here: a sweep's predictions come out of one
batched replay / capacity search as arrays (one entry per trace x config),
so `evaluate_columns` scores whole columns at once and `evaluate(jobs)` is
the reference's per-job entry point expressed through it.  The JSON
document is identical to the reference's (same rows, same aggregate, same
floating-point operations: Python int division for the relative error,
statistics.median / statistics.fmean for the aggregates).
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from .errors import EmptyInput, ZeroSize

QUADRANT_THRESHOLD = 0.2       # metrics.py:28 -- both quadrant axes
W_PROBABILITY, W_ERROR = 0.7, 0.3  # metrics.py:31-32 -- performance score


class Quadrant(Enum):
    OPTIMAL = "optimal"
    UNDERESTIMATION = "underestimation"
    OVERESTIMATION = "overestimation"
    WORST = "worst"


def predict_oom(predicted_peak: int, capacity: int) -> bool:
    """A job is predicted to OOM when its peak strictly exceeds capacity."""
    if predicted_peak <= 0 or capacity <= 0:
        raise ValueError("predicted_peak and capacity must be positive")
    return predicted_peak > capacity


@dataclass(frozen=True)
class ValidationRecord:
    """One measured run (metrics.py:37-68): round 1 unrestricted, round 2
    capped at the prediction."""

    config_id: str
    round_no: int
    device: int
    estimator: str
    actual_peak: int
    actual_oom: bool

    def __post_init__(self):
        if self.round_no not in (1, 2):
            raise ValueError(f"round must be 1 or 2, got {self.round_no}")
        if self.actual_peak < 0:
            raise ValueError("actual_peak must be >= 0")

    @classmethod
    def from_json_dict(cls, raw: dict) -> "ValidationRecord":
        return cls(str(raw["config_id"]), int(raw["round"]),
                   int(raw.get("device", 0)), str(raw.get("estimator", "")),
                   int(raw["actual_peak"]), bool(raw["actual_oom"]))

    def to_json_dict(self) -> dict:
        return {"config_id": self.config_id, "round": self.round_no,
                "device": self.device, "estimator": self.estimator,
                "actual_peak": self.actual_peak, "actual_oom": self.actual_oom}


@dataclass(frozen=True)
class MetricSet:
    failure_probability: float
    median_error: float
    performance_score: float
    quadrant: Quadrant
    run_count: int
    avg_memory_saved: float | None = None

    def to_json_dict(self) -> dict:
        d = {k: getattr(self, k) for k in (
            "failure_probability", "median_error", "performance_score")}
        d.update(quadrant=self.quadrant.value, run_count=self.run_count,
                 avg_memory_saved=self.avg_memory_saved)
        return d


@dataclass(frozen=True)
class EvalJob:
    config_id: str
    predicted_peak: int
    capacity: int
    oom_predicted: bool
    round1: ValidationRecord
    round2: ValidationRecord | None = None


def correctness_round1(predicted: bool, actual: bool) -> bool:
    return predicted == actual


def correctness_round2(c1: bool, oom1: bool, oom2: bool) -> bool:
    # a correct round 1 that either survives the capped re-run or was
    # rightly rejected outright (metrics.py:102-110)
    return c1 and (oom1 or not oom2)


def relative_error(predicted: int, actual: int) -> float:
    if actual <= 0:
        raise ZeroSize(f"actual peak must be positive, got {actual}")
    return abs(predicted - actual) / actual


def quadrant(p: float, median_error: float) -> Quadrant:
    over_p = p >= QUADRANT_THRESHOLD
    over_e = median_error >= QUADRANT_THRESHOLD
    return ((Quadrant.OPTIMAL, Quadrant.OVERESTIMATION),
            (Quadrant.UNDERESTIMATION, Quadrant.WORST))[over_p][over_e]


def memory_saved(capacity: int, predicted_peak: int, c1: bool, oom1: bool,
                 oom2: bool) -> int:
    # rejecting an impossible job saves the device; a correct prediction
    # whose capped re-run survives saves the headroom; anything else wastes
    # the device (metrics.py:160-174)
    if not c1:
        return -capacity
    if oom1:
        return capacity
    return capacity - predicted_peak if not oom2 else -capacity


def avg_memory_saved(savings: list[int]) -> float:
    if not savings:
        raise EmptyInput("no savings to average")
    return statistics.fmean(savings)


def _metric_set(n: int, n_correct: int, errors: list, savings: list) -> MetricSet:
    p = (n - n_correct) / n
    med = statistics.median(errors) if errors else 0.0
    return MetricSet(failure_probability=p, median_error=med,
                     performance_score=W_PROBABILITY * p + W_ERROR * med,
                     quadrant=quadrant(p, med), run_count=n,
                     avg_memory_saved=statistics.fmean(savings) if savings else None)


def aggregate(records: list[tuple[bool, float]]) -> MetricSet:
    """Per-run (correct, error) pairs -> MetricSet (metrics.py:119-137)."""
    if not records:
        raise EmptyInput("no records to aggregate")
    ms = _metric_set(len(records), sum(1 for c, _ in records if c),
                     [e for _, e in records], [])
    return MetricSet(ms.failure_probability, ms.median_error,
                     ms.performance_score, ms.quadrant, ms.run_count)


def evaluate_columns(config_ids: Sequence, predicted_peak, capacity,
                     oom_predicted, actual_peak, actual_oom,
                     actual_oom2=None) -> dict:
    """Score a sweep given as columns (one entry per job); returns the
    reference's evaluate() document.  `actual_oom2` is the capped re-run's
    verdict (None / False where there was no round 2)."""
    n = len(config_ids)
    if n == 0:
        raise EmptyInput("no jobs to evaluate")
    pred = np.array([int(x) for x in predicted_peak], dtype=object)
    cap = np.array([int(x) for x in capacity], dtype=object)
    act = np.array([int(x) for x in actual_peak], dtype=object)
    opred = np.asarray(oom_predicted, dtype=bool)
    oom1 = np.asarray(actual_oom, dtype=bool)
    oom2 = (np.zeros(n, dtype=bool) if actual_oom2 is None
            else np.asarray(actual_oom2, dtype=bool))
    c1 = opred == oom1
    c2 = c1 & (oom1 | ~oom2)
    has_err = act > 0
    has_cap = cap > 0
    # exact Python-int arithmetic per element, as the reference does
    err = [abs(p - a) / a if h else None for p, a, h in zip(pred, act, has_err)]
    saved = [(-k if not ok else k if o1 else (k - p if not o2 else -k)) if hc
             else None
             for p, k, ok, o1, o2, hc in zip(pred, cap, c1, oom1, oom2, has_cap)]
    rows = [{"config_id": cid, "predicted_peak": int(p), "actual_peak": int(a),
             "oom_predicted": bool(op), "actual_oom": bool(o1),
             "correctness_r1": bool(x1), "correctness_r2": bool(x2),
             "relative_error": e, "memory_saved": None if s is None else int(s)}
            for cid, p, a, op, o1, x1, x2, e, s in
            zip(config_ids, pred, act, opred, oom1, c1, c2, err, saved)]
    ms = _metric_set(n, int(c1.sum()), [e for e in err if e is not None],
                     [s for s in saved if s is not None])
    return {"jobs": rows, "aggregate": ms.to_json_dict()}


def evaluate(jobs: list[EvalJob]) -> dict:
    """metrics.py:196-241 over EvalJob objects."""
    if not jobs:
        raise EmptyInput("no jobs to evaluate")
    return evaluate_columns(
        [j.config_id for j in jobs], [j.predicted_peak for j in jobs],
        [j.capacity for j in jobs], [j.oom_predicted for j in jobs],
        [j.round1.actual_peak for j in jobs], [j.round1.actual_oom for j in jobs],
        [j.round2.actual_oom if j.round2 is not None else False for j in jobs])


def evaluate_sweep(results: np.ndarray, capacity, actual_peak, actual_oom,
                   actual_oom2=None, config_ids=None, initial_memory=0) -> dict:
    """Evaluate a batched sweep straight from the engine's per-trace result
    records (pm_result_t, e.g. DeviceBatch.results() or the `unbounded`
    records of a capacity search): prediction = peak_reserved, verdict =
    predict_oom(initial + peak, capacity) for a finite capacity, as
    estimator.py:155-158 forms them."""
    n = len(results)
    cap = np.broadcast_to(np.asarray(capacity, dtype=np.int64), (n,))
    peak = results["peak_reserved"].astype(np.int64)
    oom = [(bool(r["status"] == 1) or (c > 0 and p > 0 and initial_memory + p > c))
           for r, p, c in zip(results, peak.tolist(), cap.tolist())]
    ids = config_ids if config_ids is not None else [str(i) for i in range(n)]
    return evaluate_columns(ids, peak.tolist(), cap.tolist(), oom, actual_peak,
                            actual_oom, actual_oom2)
