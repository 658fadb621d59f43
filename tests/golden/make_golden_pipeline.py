"""Golden vectors for the analysis -> link -> orchestration -> estimate path.

Run where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_pipeline.py

Inputs: the reference's three committed fixtures (copied gzip-compressed to
tests/golden/traces/ so the GPU box has them), traces from
oracle/tracegen.py (regenerated from their seeds at test time), and the
hand-laid two-iteration trace of the reference's conftest
(pkg/tests/conftest.py:50-89), restated in tests/pipeline_cases.py.
Outputs: digests of every intermediate view the reference exposes, plus the
byte-exact estimate report.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import logging
import shutil
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
logging.disable(logging.WARNING)

from peakmem.trace import SidecarConfig, load_sidecar, parse_trace  # noqa: E402

import peakmem  # noqa: E402
from pipeline_cases import CASES, case_records, views as _views  # noqa: E402


def views(bundle):
    return _views(peakmem, bundle)


FIXTURES = Path("/root/reference/pkg/tests/fixtures")


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True,
                                     separators=(",", ":")).encode()).hexdigest()


def main():
    gold = {}
    for name in ("tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"):
        src = FIXTURES / name
        dst = HERE / "traces"
        with open(src / "trace.json", "rb") as f, \
                gzip.open(dst / f"{name}.trace.json.gz", "wb", compresslevel=9) as g:
            shutil.copyfileobj(f, g)
        shutil.copy(src / "sidecar.json", dst / f"{name}.sidecar.json")
        bundle = parse_trace(str(src / "trace.json"),
                             sidecar=load_sidecar(str(src / "sidecar.json")))
        g = views(bundle)
        g["golden_report"] = (src / "golden_report.json").read_text()
        gold[name] = g
    for case in CASES:
        recs, side = case_records(case)
        d = tempfile.mkdtemp()
        p = Path(d) / "t.json"
        p.write_text(json.dumps({"traceEvents": recs}))
        sc = None if side is None else SidecarConfig(
            param_sizes=tuple(side["param_sizes"]),
            batch_bytes=tuple(side["batch_bytes"]),
            optimizer_name=side["optimizer"],
            device_capacity=side.get("device_capacity_bytes", 0),
            initial_memory=side.get("initial_memory_bytes", 0))
        gold[case["name"]] = views(parse_trace(str(p), sidecar=sc))
    (HERE / "pipeline_golden.json").write_text(json.dumps(gold, indent=0) + "\n")
    print("wrote", len(gold), "cases")


if __name__ == "__main__":
    main()
