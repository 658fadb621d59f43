"""GPU parity of the analysis -> link -> orchestration -> estimate path.

Every case is compared with golden vectors produced by the reference itself
(tests/golden/make_golden_pipeline.py): normalized events, layer tree with
per-layer forward / backward ops and retained / temporary blocks (the
event -> operator -> layer linkage), operator roots, markers, blocks with
roles, request sequences for 1-3 iterations (incl. cloning), the blocks'
roles / lifetimes after orchestration, and the byte-exact estimate reports
(three allocator configurations).
"""

from __future__ import annotations

import gzip
import json
import logging
from pathlib import Path

import pytest

import paper_2504_03887_b200 as api
from conftest import GOLDEN, golden
from pipeline_cases import CASES, case_records, views

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]
logging.disable(logging.WARNING)

FIXTURES = ["tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"]


def fixture_bundle(name, tmp_path):
    trace = tmp_path / f"{name}.json"
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        trace.write_bytes(f.read())
    side = api.load_sidecar(GOLDEN / "traces" / f"{name}.sidecar.json")
    return api.parse_trace(trace, sidecar=side)


def case_bundle(case, tmp_path):
    recs, side = case_records(case)
    p = tmp_path / f"{case['name']}.json"
    p.write_text(json.dumps({"traceEvents": recs}))
    sc = api.SidecarConfig(param_sizes=tuple(side["param_sizes"]),
                           batch_bytes=tuple(side["batch_bytes"]),
                           optimizer_name=side["optimizer"],
                           device_capacity=side.get("device_capacity_bytes", 0),
                           initial_memory=side.get("initial_memory_bytes", 0))
    return api.parse_trace(p, sidecar=sc)


def compare(got: dict, want: dict):
    for key in want:
        if key == "golden_report":
            continue
        assert got[key] == want[key], key


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_pipeline_matches_reference(name, tmp_path):
    bundle = fixture_bundle(name, tmp_path)
    want = golden("pipeline_golden.json")[name]
    compare(views(api, bundle), want)
    # the committed golden report, byte for byte (test_acceptance.py:347-359)
    assert api.PeakMemoryEstimator().estimate(bundle).canonical_json() == \
        want["golden_report"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_generated_pipeline_matches_reference(case, tmp_path):
    bundle = case_bundle(case, tmp_path)
    compare(views(api, bundle), golden("pipeline_golden.json")[case["name"]])


@pytest.mark.parametrize("seed,kw", [
    (101, {"layers": 160, "leaves": 4, "iterations": 3}),
    (102, {"layers": 80, "leaves": 6, "iterations": 1, "optimizer": "sgd"}),
    (103, {"layers": 120, "leaves": 3, "iterations": 4, "zero_grad": "pre-backward"}),
])
def test_large_generated_pipeline_vs_oracle(seed, kw, tmp_path):
    """Traces too large for committed goldens: GPU vs the pinned oracle."""
    from oracle import pipeline as op
    case = {"name": f"large_{seed}", "seed": seed, "kw": kw}
    records, side = case_records(case)
    bundle = case_bundle(case, tmp_path)
    events = op.normalize(records)
    for it in (1, 2, 3):
        want = op.build_sequence(events, side, it)
        got = api.build_sequence(api.analyze(bundle), iterations=it)
        assert [(r.kind.value, r.block_id, r.size, r.virtual_ts)
                for r in got.requests] == want, it


def test_c5_style_trace_vs_oracle():
    """SURVEY C5 shape (one long trace) at 2e5 events: GPU vs oracle."""
    from oracle import pipeline as op
    from paper_2504_03887_b200 import synth_events
    b = synth_events.generate(6000, iterations=2)
    assert len(b) > 150_000
    recs = b.to_json_dict()["traceEvents"]
    side = {"param_sizes": list(b.metadata.param_sizes),
            "batch_bytes": list(b.metadata.batch_bytes)}
    want = op.build_sequence(op.normalize(recs), side, 2)
    got = api.build_sequence(api.analyze(b), iterations=2)
    assert [(r.kind.value, r.block_id, r.size, r.virtual_ts)
            for r in got.requests] == want


def test_c5_1e6_events_vs_oracle():
    """GPU-vs-oracle pipeline parity at 10^6 events (one long
    C5-style trace, 2 iterations): the orchestrated request sequence and its
    replay (every result field) equal the CPU oracle's."""
    import numpy as np
    from oracle import pipeline as op
    from oracle import replay as oracle_replay
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.estimator import replay_sequence
    b = synth_events.generate(36000, iterations=2)
    assert len(b) > 1_000_000
    recs = b.to_json_dict()["traceEvents"]
    side = {"param_sizes": list(b.metadata.param_sizes),
            "batch_bytes": list(b.metadata.batch_bytes)}
    want = op.build_sequence(op.normalize(recs), side, 2)
    got = api.build_sequence(api.analyze(b), iterations=2)
    assert [(r.kind.value, r.block_id, r.size, r.virtual_ts)
            for r in got.requests] == want
    res = replay_sequence(got, AllocatorConfig(), timeline=False)
    offs = np.array([0, len(got.packed)], dtype=np.int64)
    ref, _ = oracle_replay.replay_batch(got.packed, offs, cfg_record(AllocatorConfig()))
    assert res.peak_reserved == int(ref[0]["peak_reserved"])
    assert res.peak_allocated == int(ref[0]["peak_allocated"])
    assert res.final_reserved == int(ref[0]["final_reserved"])
    assert res.n_segments_peak == int(ref[0]["n_segments_peak"])
