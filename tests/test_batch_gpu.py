"""GPU: the batched, device-resident pipeline (pm_pipeline_batch,
paper_2504_03887_b200/batch.py) against the reference's goldens and the
per-trace path.

* every pipeline golden case (3 fixtures, 16 generated traces, the
  reference conftest's hand-laid iterations) and the two real captures in
  ONE estimate_many call per configuration: reports byte-identical to the
  reference's, failing traces raising the reference's error class
  (tests/golden/make_golden_pipeline.py, make_golden_captures.py);
* build_sequences == build_sequence(analyze(b)) record for record, for 1-3
  iterations, in mixed batches (repeated traces, failing traces between good
  ones, a trace with no instants / no layers);
* a batch whose traces share python ids, addresses, sequence numbers and
  timestamps (copies of one trace) gives each copy the single-trace answer.
"""

from __future__ import annotations

import gzip
import json
import logging

import numpy as np
import pytest

import paper_2504_03887_b200 as api
from conftest import GOLDEN, golden
from paper_2504_03887_b200.batch import build_sequences
from pipeline_cases import CASES
from test_pipeline_gpu import FIXTURES, case_bundle, fixture_bundle

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]
logging.disable(logging.WARNING)

CONFIGS = (("default", {}), ("cap", {"device_capacity": 64 << 20}),
           ("split", {"max_split_size": 32 << 20, "iterations": 3}))
CAPTURES = ["resnet18_bs32_224", "gpt2_bs8_s128"]


def capture_bundle(name, tmp_path):
    trace = tmp_path / f"{name}.json"
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        trace.write_bytes(f.read())
    side = api.load_sidecar(GOLDEN / "traces" / f"{name}.sidecar.json")
    return api.parse_trace(trace, sidecar=side)


@pytest.fixture(scope="module")
def all_bundles(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("batch")
    names, bundles, wants = [], [], []
    g = golden("pipeline_golden.json")
    for name in FIXTURES:
        names.append(name)
        bundles.append(fixture_bundle(name, tmp))
        wants.append(g[name])
    for case in CASES:
        names.append(case["name"])
        bundles.append(case_bundle(case, tmp))
        wants.append(g[case["name"]])
    cg = golden("captures_golden.json")
    for name in CAPTURES:
        names.append(name)
        bundles.append(capture_bundle(name, tmp))
        wants.append(cg[name])
    return names, bundles, wants


@pytest.mark.parametrize("cfg,kw", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_estimate_many_matches_reference_reports(all_bundles, cfg, kw):
    names, bundles, wants = all_bundles
    got = api.PeakMemoryEstimator(**kw).estimate_many(bundles, return_exceptions=True)
    assert len(got) == len(bundles)
    for name, g, want in zip(names, got, wants):
        w = want[f"report_{cfg}"]
        if isinstance(w, dict):  # the reference raised
            assert isinstance(g, Exception), name
            assert type(g).__name__ == w["error"], (name, g)
        else:
            assert not isinstance(g, Exception), (name, g)
            assert g.canonical_json() == w, name


def test_estimate_many_raises_first_error(all_bundles):
    """A loop over estimate raises the first failing trace's error: a trace
    without a sidecar (MissingBatchBytes, orchestration.py:246-249) between
    good ones; with return_exceptions only that slot holds it."""
    import copy
    from paper_2504_03887_b200.errors import MissingBatchBytes
    names, bundles, wants = all_bundles
    bare = copy.copy(bundles[0])
    bare.metadata = None
    batch = [bundles[1], bare, bundles[2]]
    with pytest.raises(MissingBatchBytes):
        api.PeakMemoryEstimator().estimate_many(batch)
    got = api.PeakMemoryEstimator().estimate_many(batch, return_exceptions=True)
    assert isinstance(got[1], MissingBatchBytes)
    assert got[0].canonical_json() == wants[1]["report_default"]
    assert got[2].canonical_json() == wants[2]["report_default"]


def _single(bundle, it):
    try:
        return api.build_sequence(api.analyze(bundle), iterations=it).packed
    except Exception as exc:  # noqa: BLE001
        return exc


@pytest.mark.parametrize("it", [1, 2, 3])
def test_build_sequences_equals_per_trace(all_bundles, it):
    names, bundles, _ = all_bundles
    # repeats (identical ids / addresses / seqs / times in one batch) and a
    # shuffled order
    rng = np.random.default_rng(it)
    order = list(range(len(bundles))) + [0, 5, 5, len(bundles) - 1]
    rng.shuffle(order)
    batch = build_sequences([bundles[i] for i in order], iterations=it)
    for k, i in enumerate(order):
        want = _single(bundles[i], it)
        if isinstance(want, Exception):
            assert type(batch.errors[k]) is type(want), names[i]
            continue
        assert batch.errors[k] is None, (names[i], batch.errors[k])
        got = batch.packed(k)
        assert len(got) == len(want), names[i]
        assert (got == want).all(), names[i]


def test_breakdown_matches_sequence(all_bundles):
    names, bundles, _ = all_bundles
    batch = build_sequences(bundles, iterations=2)
    for k, b in enumerate(bundles):
        if batch.errors[k] is not None:
            continue
        seq = api.build_sequence(api.analyze(b), iterations=2)
        assert batch.breakdown(k) == seq.breakdown(), names[k]
        assert int(batch.n_model[k]) == seq._arrays["n_model"], names[k]


def test_single_trace_batch_and_large_trace():
    """B = 1 on a C5-style trace of ~1.7e5 events equals the per-trace path."""
    from paper_2504_03887_b200 import synth_events
    b = synth_events.generate(6000, iterations=2)
    want = api.build_sequence(api.analyze(b), iterations=2).packed
    batch = build_sequences([b], iterations=2)
    assert batch.errors == [None]
    assert (batch.packed(0) == want).all()
    # and as one of several copies
    batch = build_sequences([b, b, b], iterations=2)
    for k in range(3):
        assert (batch.packed(k) == want).all()


def test_estimate_many_validate_flag(all_bundles):
    names, bundles, wants = all_bundles
    pick = [i for i, w in enumerate(wants) if not isinstance(w["report_default"], dict)][:4]
    got = api.PeakMemoryEstimator(validate=True).estimate_many([bundles[i] for i in pick])
    for i, g in zip(pick, got):
        assert g.canonical_json() == wants[i]["report_default"], names[i]


@pytest.mark.parametrize("it", [1, 2, 3])
def test_lazy_build_sequence_equals_viewed_path(all_bundles, it):
    """build_sequence on an analyzed trace whose views were never asked for
    (pm_pipeline_batch with views) == the per-stage path (pm_link +
    pm_orchestrate, taken once a view exists): the request sequence, its
    phase tags and boundaries, and the analyzed blocks mutated in place."""
    names, bundles, _ = all_bundles
    for name, b in zip(names, bundles):
        lazy = api.analyze(b)
        viewed = api.analyze(b)
        _ = viewed.blocks  # materialise: the per-stage path
        try:
            s_viewed = api.build_sequence(viewed, iterations=it)
        except Exception as exc:  # noqa: BLE001
            with pytest.raises(type(exc)):
                api.build_sequence(lazy, iterations=it)
            continue
        s_lazy = api.build_sequence(lazy, iterations=it)
        assert s_lazy.to_json_dict() == s_viewed.to_json_dict(), name
        assert (s_lazy.packed == s_viewed.packed).all(), name
        assert [(x.block_id, x.free_time, x.role) for x in lazy.blocks] == \
            [(x.block_id, x.free_time, x.role) for x in viewed.blocks], name
