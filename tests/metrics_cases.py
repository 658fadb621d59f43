"""Seeded evaluation-job batches shared by tests/golden/make_golden_metrics.py
(the reference scores them) and tests/test_metrics.py (the engine does)."""

import random

GIB = 1 << 30


def _job(rng, i):
    actual = rng.choice([0, rng.randint(1, 80 * GIB)])
    pred = max(1, int(actual * rng.uniform(0.6, 1.5))) if actual else rng.randint(1, 80 * GIB)
    cap = rng.choice([0, 24 * GIB, 40 * GIB, 80 * GIB])
    oom1 = rng.random() < 0.3
    r2 = None
    if rng.random() < 0.7:
        r2 = {"config_id": f"c{i}", "round_no": 2, "device": 1, "estimator": "xmem",
              "actual_peak": rng.randint(0, 80 * GIB), "actual_oom": rng.random() < 0.3}
    return {"config_id": f"c{i}", "predicted_peak": pred, "capacity": cap,
            "oom_predicted": (pred > cap) if cap else rng.random() < 0.2,
            "round1": {"config_id": f"c{i}", "round_no": 1, "device": 0,
                       "estimator": "xmem", "actual_peak": actual,
                       "actual_oom": oom1},
            "round2": r2}


def batches():
    rng = random.Random(20250403)
    out = []
    for n in (1, 2, 3, 10, 57, 400):
        out.append([_job(rng, i) for i in range(n)])
    return out
