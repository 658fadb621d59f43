"""CPU: pin the pipeline oracle (oracle/pipeline.py) to the reference's
goldens (tests/golden/pipeline_golden.json): request lists for 1-3
iterations on every golden trace, including the committed fixtures."""

from __future__ import annotations

import gzip
import json

import pytest

from conftest import GOLDEN, golden
from oracle import pipeline as op
from pipeline_cases import CASES, case_records, digest

FIXTURES = ["tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"]


def check(name, records, side):
    want = golden("pipeline_golden.json")[name]
    events = op.normalize(records)
    assert len(events) == want["n_events"]
    for it in (1, 2, 3):
        w = want[f"seq{it}"]
        if "error" in w:
            with pytest.raises(ValueError):
                op.build_sequence(events, side, it)
            continue
        seq = op.build_sequence(events, side, it)
        assert len(seq) == w["n"]
        assert digest(op.request_digest_rows(seq)) == w["req_sha256"], (name, it)


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_fixture_sequences(name):
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        records = json.loads(f.read())["traceEvents"]
    side = json.loads((GOLDEN / "traces" / f"{name}.sidecar.json").read_text())
    check(name, records, side)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_generated_sequences(case):
    records, side = case_records(case)
    check(case["name"], records, side)
