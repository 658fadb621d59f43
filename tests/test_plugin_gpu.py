"""GPU: the engine bound into the reference's own pipeline via plugin.install().

Needs the reference package: `baseline/_ref` (pip-installed copy of the
reference, git-ignored, shipped to the GPU box) or /root/reference.
"""

from __future__ import annotations

import gzip
import sys
from pathlib import Path

import pytest

from conftest import GOLDEN, REPO, golden
from replay_cases import corpus

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


@pytest.fixture(scope="module")
def peakmem():
    for cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "peakmem").exists():
            sys.path.insert(0, str(cand))
            break
    mod = pytest.importorskip("peakmem")
    from paper_2504_03887_b200 import plugin
    plugin.install(pipeline=True)
    yield mod
    plugin.uninstall()


def test_reference_estimator_runs_on_gpu_and_matches_golden(peakmem, tmp_path):
    import peakmem.estimator as est
    assert est.replay.__module__.startswith("paper_2504_03887_b200")
    for name in ("tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"):
        trace = tmp_path / f"{name}.json"
        with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
            trace.write_bytes(f.read())
        side = peakmem.load_sidecar(str(GOLDEN / "traces" / f"{name}.sidecar.json"))
        bundle = peakmem.parse_trace(str(trace), sidecar=side)
        report = peakmem.PeakMemoryEstimator().estimate(bundle)
        assert report.canonical_json() == \
            golden("pipeline_golden.json")[name]["golden_report"]


def test_reference_replay_api_on_gpu(peakmem):
    from peakmem.allocator import AllocatorConfig, replay
    from peakmem.errors import MalformedSequence
    cases = corpus("corpus_seed1000")[:100]
    gold = golden("replay_corpus_seed1000.json")["cases"]
    for (seq, params), g in zip(cases, gold):
        cfg = AllocatorConfig(device_capacity=params["capacity"],
                              max_split_size=params["max_split_size"])
        out = replay(seq, cfg)
        assert type(out).__module__ == "peakmem.allocator"
        assert out.peak_reserved == g["peak_reserved"]
        assert out.oom_seq_no == g["oom_seq_no"]
    with pytest.raises(MalformedSequence):
        replay([{"seq_no": 0, "kind": "free", "block_id": 1}])


def test_reference_module_path_analyze_then_build_sequence(peakmem, tmp_path):
    """peakmem.orchestration.build_sequence(peakmem.orchestration.analyze(b))
    -- the reference's own public path -- runs on the engine end to end and
    yields the reference's sequence (the aliases are rebound together)."""
    import peakmem.orchestration as orch
    from peakmem.allocator import replay
    for name in ("tiny_mlp_sgd", "tiny_mlp_adam"):
        trace = tmp_path / f"{name}.json"
        with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
            trace.write_bytes(f.read())
        side = peakmem.load_sidecar(str(GOLDEN / "traces" / f"{name}.sidecar.json"))
        bundle = peakmem.parse_trace(str(trace), sidecar=side)
        for build, analyze in ((orch.build_sequence, orch.analyze),
                               (peakmem.build_sequence, peakmem.analyze)):
            seq = build(analyze(bundle), iterations=2)
            assert type(seq).__module__ == "peakmem.orchestration"
            assert all(type(r.kind) is orch.RequestKind for r in seq.requests)
            gold = golden("replay_fixture_sequences.json")[name]
            assert seq.replay_records() == gold["records"]
            assert replay(seq.replay_records()).peak_reserved == \
                gold["result"]["peak_reserved"]


def test_reference_built_analyzed_trace_still_accepted(peakmem, tmp_path):
    """An AnalyzedTrace built by the reference before install() goes to the
    reference's own build_sequence (its enums), not the engine's."""
    from paper_2504_03887_b200 import plugin
    import peakmem.orchestration as orch
    name = "tiny_mlp_sgd"
    trace = tmp_path / f"{name}.json"
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        trace.write_bytes(f.read())
    side = peakmem.load_sidecar(str(GOLDEN / "traces" / f"{name}.sidecar.json"))
    bundle = peakmem.parse_trace(str(trace), sidecar=side)
    plugin.uninstall()
    try:
        analyzed = orch.analyze(bundle)
    finally:
        plugin.install(pipeline=True)
    seq = orch.build_sequence(analyzed, iterations=2)
    assert seq.replay_records() == \
        golden("replay_fixture_sequences.json")[name]["records"]
