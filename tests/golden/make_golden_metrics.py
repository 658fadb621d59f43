"""Goldens for the evaluation metrics (reference metrics.py:98-241).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_metrics.py

Random job batches (seeded; edge cases: zero actual peak, zero capacity,
missing round 2, OOM both ways, even / odd counts) scored by the reference's
evaluate(); tests/test_metrics.py regenerates the same jobs and compares the
documents exactly.
"""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from peakmem.metrics import EvalJob, ValidationRecord, aggregate, evaluate  # noqa: E402

from metrics_cases import batches  # noqa: E402


def main():
    out = []
    for jobs in batches():
        ev = evaluate([EvalJob(j["config_id"], j["predicted_peak"], j["capacity"],
                               j["oom_predicted"],
                               ValidationRecord(**j["round1"]),
                               ValidationRecord(**j["round2"]) if j["round2"] else None)
                       for j in jobs])
        agg = aggregate([(r["correctness_r1"], r["relative_error"] or 0.0)
                         for r in ev["jobs"]]).to_json_dict()
        out.append({"evaluate": ev, "aggregate": agg})
    (HERE / "metrics_golden.json").write_text(json.dumps(out, indent=0) + "\n")
    print(len(out), "batches")


if __name__ == "__main__":
    main()
