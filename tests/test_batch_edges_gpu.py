"""GPU: pm_pipeline_batch on batches that mix failing and degenerate traces
with good ones.  Every trace's outcome (the error build_sequence raises, or
its request sequence) must be what the per-trace path gives for it alone --
the per-trace path is pinned to the reference's goldens elsewhere
(tests/test_pipeline_gpu.py) -- and no trace may leak into another."""

from __future__ import annotations

import json

import pytest

import paper_2504_03887_b200 as api
from paper_2504_03887_b200.batch import build_sequences
from pipeline_cases import case_records, ev, iteration_records

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def bundle_of(recs, side, tmp_path, name):
    p = tmp_path / f"{name}.json"
    p.write_text(json.dumps({"traceEvents": recs}))
    sc = None if side is None else api.SidecarConfig(
        param_sizes=tuple(side["param_sizes"]), batch_bytes=tuple(side["batch_bytes"]),
        optimizer_name=side.get("optimizer", "sgd"))
    return api.parse_trace(p, sidecar=sc)


SIDE = {"param_sizes": [400], "batch_bytes": [128, 64], "optimizer": "sgd"}


def cases():
    two = iteration_records(0, 0, with_grad_free_at=1010) + iteration_records(1, 1000)
    out = {
        "conftest": (two, SIDE),
        "no_instants": ([r for r in two if r["cat"] != "cpu_instant_event"], SIDE),
        "no_layers": ([r for r in two if r["cat"] != "python_function"], SIDE),
        "no_ops": ([r for r in two if r["cat"] != "cpu_op"], SIDE),
        "no_markers": ([r for r in two if r["cat"] != "user_annotation"], SIDE),
        "no_batch_bytes": (two, {**SIDE, "batch_bytes": []}),
        "no_sidecar": (two, None),
        "cyclic": (two + [
            ev("python_function", "nn.Module: Loop", 5, 3, **{"Python id": 9050,
                                                              "Python parent id": 9051}),
            ev("python_function", "helper", 4, 6, **{"Python id": 9051,
                                                      "Python parent id": 9050})], SIDE),
        "gen_s1": case_records({"name": "gen_s1", "seed": 1}),
        "gen_s7_wide": case_records({"name": "g7", "seed": 7,
                                     "kw": {"layers": 2, "leaves": 12}}),
    }
    return out


def _single(b, it):
    try:
        return api.build_sequence(api.analyze(b), iterations=it).packed
    except Exception as exc:  # noqa: BLE001 -- compared by class
        return exc


@pytest.mark.parametrize("it", [1, 2, 3])
def test_mixed_batch_matches_each_trace_alone(tmp_path, it):
    cs = cases()
    names = list(cs) + ["gen_s1", "cyclic", "conftest"]  # repeats
    bundles = {n: bundle_of(r, s, tmp_path, n) for n, (r, s) in cs.items()}
    batch = build_sequences([bundles[n] for n in names], iterations=it)
    seen_error = set()
    for k, n in enumerate(names):
        want = _single(bundles[n], it)
        got_err = batch.errors[k]
        if isinstance(want, Exception):
            assert type(got_err) is type(want), (n, got_err, want)
            seen_error.add(type(want).__name__)
        else:
            assert got_err is None, (n, got_err)
            got = batch.packed(k)
            assert len(got) == len(want) and (got == want).all(), n
    # the degenerate cases really exercise the error paths
    assert {"CyclicParentLink", "MissingBatchBytes"} <= seen_error
