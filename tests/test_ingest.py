"""Native trace reader and config digest (csrc/ingest.cpp)
against the Python restatement of the reference's rules (trace.py:174-238,
estimator.py:189-202).  CPU only: the reader and the digest are host code.

Bar: identical columns (bit-exact fp64 ts/dur, int64 fields, names) or the
native reader declines (UNSUPPORTED) so the Python reader applies the
reference's exact errors; identical SHA-256 digests."""

from __future__ import annotations

import gzip
import json
import logging
import random

import numpy as np
import pytest

from conftest import GOLDEN
from pipeline_cases import CASES, case_records
from paper_2504_03887_b200 import _ingest
from paper_2504_03887_b200.errors import EmptyTrace, MalformedTrace
from paper_2504_03887_b200.estimator import PeakMemoryEstimator
from paper_2504_03887_b200.trace import (SidecarConfig, TraceBundle,
                                         _INT_FIELDS, collect_records,
                                         load_sidecar)

logging.disable(logging.WARNING)
CAPTURES = ["tiny_mlp_adam", "tiny_mlp_sgd", "tiny_mlp_sgd_pregrad",
            "resnet18_bs32_224", "gpt2_bs8_s128"]


def python_columns(text: str, strict=False):
    raw = json.loads(text)
    records = raw["traceEvents"] if isinstance(raw, dict) else raw
    return collect_records(records, "", strict)


def assert_same(native, text, strict=False):
    ts, dur, cat, ints, names = python_columns(text, strict)
    nts, ndur, ncat, nints, nnames, _ = native
    assert nts.tobytes() == ts.tobytes()
    assert ndur.tobytes() == dur.tobytes()
    assert np.array_equal(ncat, cat)
    for k, f in enumerate(_INT_FIELDS):
        assert np.array_equal(nints[k], ints[f]), f
    assert nnames == names


def check_text(text: str, strict=False):
    """Native accepts -> identical to Python; Python errors -> native declined."""
    got = _ingest.parse_json(text.encode("utf-8"), strict)
    try:
        python_columns(text, strict)
    except EmptyTrace:
        assert got in (_ingest.EMPTY, _ingest.UNSUPPORTED), text[:200]
        return "empty"
    except (MalformedTrace, json.JSONDecodeError, TypeError, ValueError,
            AttributeError, KeyError):
        assert got == _ingest.UNSUPPORTED, text[:200]
        return "error"
    if isinstance(got, int):
        assert got == _ingest.UNSUPPORTED
        return "declined"
    assert_same(got, text, strict)
    return "native"


def capture_text(name):
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        return f.read().decode("utf-8")


@pytest.mark.parametrize("name", CAPTURES)
def test_captures_native_equals_python(name):
    assert check_text(capture_text(name)) == "native"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_generated_native_equals_python(case):
    recs = case_records(case)
    recs = recs[0] if isinstance(recs, tuple) else recs
    for text in (json.dumps({"traceEvents": recs}), json.dumps(recs, indent=1)):
        assert check_text(text) == "native"


def _fuzz_value(rng: random.Random):
    return rng.choice([
        0, 1, -1, 7, 2**40 + 3, -2**40, 2**62, 2**63 - 1, -2**63, 2**63, 2**64,
        1.5, -2.75, 3.0, 1e300, 1e-300, 0.1, 123456789.123, -0.0, True, False,
        None, "12", "x", [], {}, [1], {"a": 1}])


def _fuzz_record(rng: random.Random, i: int):
    cat = rng.choice(["python_function", "cpu_op", "user_annotation",
                      "cpu_instant_event", "other", "gpu_op", "kernel", None, 3,
                      ["x"]])
    rec = {}
    if rng.random() < 0.05:
        rec["ph"] = "M"
    elif rng.random() < 0.9:
        rec["ph"] = rng.choice(["X", "i", "B"])
    if rng.random() < 0.95:
        rec["cat"] = cat
    if rng.random() < 0.9:
        rec["name"] = rng.choice([f"op{i}", "nn.Module: Linear_0", "éé",
                                  "tab\tnewline\n\"q\"\\", "中文",
                                  "\U0001F600 emoji", "ctl", "", 5, None])
    if rng.random() < 0.97:
        rec["ts"] = rng.choice([i, i * 1.25, float(i) + 0.5, 10**15 + i,
                                rng.uniform(0, 1e6), _fuzz_value(rng)])
    if rng.random() < 0.8:
        rec["dur"] = rng.choice([0, 1, 2.5, 100, None, 0.0, rng.uniform(0, 50),
                                 _fuzz_value(rng)])
    args = {}
    for key in ("Python id", "Python parent id", "Sequence number", "Addr",
                "Bytes", "Total Allocated", "Total Reserved", "Other"):
        if rng.random() < 0.5:
            args[key] = rng.choice([rng.randrange(-5, 2**20), rng.randrange(1, 100),
                                    _fuzz_value(rng)])
    r = rng.random()
    if r < 0.85:
        rec["args"] = args
    elif r < 0.9:
        rec["args"] = None
    elif r < 0.95:
        rec["args"] = rng.choice([[], 0, "", "s", [1]])
    return rec


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_native_equals_python_or_declines(seed):
    rng = random.Random(seed)
    outcomes = set()
    for _ in range(12):
        n = rng.randrange(0, 30)
        recs = [_fuzz_record(rng, i) for i in range(n)]
        if rng.random() < 0.3:  # keep to the well-formed subset often
            recs = [r for r in recs if isinstance(r.get("cat"), str)]
        strict = rng.random() < 0.2
        root = {"traceEvents": recs} if rng.random() < 0.7 else recs
        text = json.dumps(root, ensure_ascii=rng.random() < 0.5,
                          indent=rng.choice([None, 1]))
        outcomes.add(check_text(text, strict))
    assert outcomes  # every text checked


def _clean_record(rng: random.Random, i: int):
    """Well-typed records: the native reader's subset (floats / bools /
    big ints in int fields, unicode names, unknown categories, drops)."""
    num = [0, 1, -1, 2**40 + 3, 2**63 - 1, -2**63 + 1, 1.5, -2.75, 3.0, 0.1, True,
           False, None, 1e18, -1e18, 7.999999]
    rec = {"ph": rng.choice(["X", "i", "M", "B"]) if rng.random() < 0.9 else "X",
           "cat": rng.choice(["python_function", "cpu_op", "user_annotation",
                              "cpu_instant_event", "other", "gpu_op"]),
           "ts": rng.choice([i, i * 1.25, 10**15 + i, rng.uniform(0, 1e6),
                             1e-300, 2.0**53 + 1, -3.5])}
    if rng.random() < 0.9:
        rec["name"] = rng.choice([f"op{i}", "éé", "tab\t\"q\"\\", "中文",
                                  "\U0001F600", "\u0001", ""])
    if rng.random() < 0.8:
        rec["dur"] = rng.choice([0, 1, 2.5, None, 0.0, False, rng.uniform(0, 50)])
    if rng.random() < 0.9:
        rec["args"] = {k: rng.choice(num + [rng.randrange(-5, 2**20)] * 4)
                       for k in ("Python id", "Python parent id", "Sequence number",
                                 "Addr", "Bytes", "Total Allocated",
                                 "Total Reserved", "Extra") if rng.random() < 0.6}
        if rng.random() < 0.1:
            rec["args"]["Nested"] = {"a": [1, {"b": None}], "c": "s"}
    if rng.random() < 0.1:
        rec["extra"] = [1, 2, {"x": "y"}]
    return rec


@pytest.mark.parametrize("seed", range(30))
def test_fuzz_clean_records_native(seed):
    rng = random.Random(1000 + seed)
    outcomes = []
    for _ in range(8):
        recs = [_clean_record(rng, i) for i in range(rng.randrange(1, 60))]
        text = json.dumps({"traceEvents": recs}, ensure_ascii=rng.random() < 0.5)
        outcomes.append(check_text(text, strict=rng.random() < 0.1))
    assert outcomes.count("native") >= 4, outcomes


@pytest.mark.parametrize("text", [
    '{"traceEvents": []}', '[]', '{"traceEvents": [{"ph": "M", "ts": 1}]}',
    '[{"cat": "cpu_instant_event", "ts": 1, "args": {"Addr": 1, "Bytes": 0}}]',
])
def test_empty(text):
    assert _ingest.parse_json(text.encode(), False) == _ingest.EMPTY


@pytest.mark.parametrize("text", [
    '{"traceEvents": [{"ts": 1.}]}', '{"traceEvents": [{"ts": .5}]}',
    '{"traceEvents": [{"ts": 01}]}', '{"traceEvents": [{"ts": 1e}]}',
    '{"traceEvents": [{"ts": NaN}]}', '{"traceEvents": [{"ts": Infinity}]}',
    '{"traceEvents": [{"ts": 1}, ]}', '{"traceEvents": [{"ts": 1}]} x',
    '{"x": 1}', '5', '"s"',
    '{"traceEvents": [{"cat": "cpu_op", "ts": 1, "args": {"Sequence number": "3"}}]}',
    '{"traceEvents": [{"name": "\\ud800", "ts": 1}]}',
])
def test_declines_outside_subset(text):
    assert _ingest.parse_json(text.encode(), False) == _ingest.UNSUPPORTED


@pytest.mark.parametrize("text", [
    '{"traceEvents": [{"ts": 1, "ts": 2}]}',
    '{"traceEvents": [{"cat": "cpu_op", "cat": "python_function", "ts": 1, '
    '"args": {"Python id": 3, "Python id": 4}}]}',
    '{"traceEvents": [{"cat": "cpu_instant_event", "ts": 1, "args": {"Addr": 1, '
    '"Bytes": 0}, "args": {"Addr": 1, "Bytes": 8}}]}',
])
def test_duplicate_keys_last_wins(text):
    assert check_text(text) == "native"


def test_parse_trace_errors_match_python_reader(tmp_path):
    from paper_2504_03887_b200.trace import parse_trace
    bad = tmp_path / "bad.json"
    bad.write_text('{"traceEvents": [{"cat": "cpu_op", "name": "a", "ts": 1, '
                   '"args": {"Sequence number": "x"}}]}')
    with pytest.raises(MalformedTrace, match="non-integer sequence number"):
        parse_trace(bad)
    empty = tmp_path / "empty.json"
    empty.write_text('{"traceEvents": []}')
    with pytest.raises(EmptyTrace):
        parse_trace(empty)
    with pytest.raises(MalformedTrace, match="not valid JSON"):
        bad.write_text("{")
        parse_trace(bad)


def _bundle_from_text(text, sidecar):
    ts, dur, cat, ints, names = python_columns(text)
    ts, dur = np.clip(ts, -2.0**60, 2.0**60), np.clip(dur, 0, 2.0**60)
    # the digest does not care about order: floor/ceil without the sort
    start = np.floor(ts).astype(np.int64)
    end = np.ceil(ts + dur).astype(np.int64)
    return TraceBundle(category=cat, start=start, duration=end - start,
                       ints=ints, names=names, metadata=sidecar)


@pytest.mark.parametrize("name", CAPTURES)
@pytest.mark.parametrize("max_split", [None, 0, 2**21])
def test_digest_native_equals_json(name, max_split):
    side = load_sidecar(GOLDEN / "traces" / f"{name}.sidecar.json")
    bundle = _bundle_from_text(capture_text(name), side)
    est = PeakMemoryEstimator(iterations=3, max_split_size=max_split)
    cap, init = 80 * 2**30, 12345
    assert _ingest.bundle_digest(bundle, side, 3, cap, init, max_split) == \
        est._digest_json(bundle, cap, init)


@pytest.mark.parametrize("seed", range(6))
def test_digest_fuzz_names_and_nulls(seed):
    rng = random.Random(seed)
    recs = [r for r in (_fuzz_record(rng, i) for i in range(200))]
    text = json.dumps({"traceEvents": recs})
    try:
        cols = python_columns(text)
    except Exception:
        recs = [r for r in recs if isinstance(r.get("cat"), str)
                and isinstance(r.get("ts"), (int, float))
                and not isinstance(r.get("ts"), bool)]
        for r in recs:
            r["args"] = {}
            r["dur"] = 1
            if not isinstance(r.get("name"), str):
                r["name"] = "n"
        text = json.dumps({"traceEvents": recs})
        cols = python_columns(text)
    if len(cols[0]) == 0:
        pytest.skip("no events survived")
    side = None if seed % 2 else SidecarConfig(
        param_sizes=(4, 8), batch_bytes=(16,), optimizer_name="Adamé\"",
        device_capacity=7, initial_memory=1)
    bundle = _bundle_from_text(text, side)
    est = PeakMemoryEstimator(iterations=2)
    assert _ingest.bundle_digest(bundle, side, 2, 1 << 34, 0, None) == \
        est._digest_json(bundle, 1 << 34, 0)


def test_digest_synthetic_name_view():
    from paper_2504_03887_b200 import synth_events
    b = synth_events.generate(leaves=50, iterations=2)
    est = PeakMemoryEstimator()
    assert _ingest.bundle_digest(b, b.metadata, 2, 1 << 36, 0, None) == \
        est._digest_json(b, 1 << 36, 0)


# ---- the parallel chunked parse of large arrays ------------------------------

def _big_records(seed, n):
    rng = random.Random(seed)
    return [_clean_record(rng, i) for i in range(n)]


@pytest.mark.parametrize("layout", ["torch", "compact", "nested_at_cut", "trailing_keys",
                                    "top_level_array"])
def test_parallel_chunks_equal_python(layout):
    # > 2 MB per document so the reader cuts the array into chunks; every
    # layout must give the sequential (Python-reader) columns: cuts at
    # record starts are taken, cuts that land inside a record or find no
    # record start fall back to the sequential parse
    recs = _big_records(77, 40_000)
    if layout == "torch":  # profiler layout: records at "\n  {"
        text = json.dumps({"schemaVersion": 1, "traceEvents": recs}, indent=2)
    elif layout == "compact":  # one line: no cut point at all
        text = json.dumps({"traceEvents": recs})
    elif layout == "nested_at_cut":  # "\n  {" inside records too
        body = ",".join("\n  {\n\"x\": \n  {\"y\": 1},\n" + json.dumps(r)[1:] for r in recs)
        text = '{"traceEvents": [' + body + "\n]}"
    elif layout == "trailing_keys":
        text = json.dumps({"traceEvents": recs, "after": [{"a": 1}] * 3000,
                           "z": {"q": 2}}, indent=2)
    else:
        text = json.dumps(recs, indent=2)
    assert len(text) > 4 << 20
    got = _ingest.parse_json(text.encode("utf-8"), False)
    assert isinstance(got, tuple), layout
    assert_same(got, text)


def test_invalid_utf8_declined_and_parse_trace_raises(tmp_path):
    from paper_2504_03887_b200.trace import parse_trace
    good = json.dumps({"traceEvents": [{"ph": "X", "cat": "cpu_op", "name": "é",
                                        "ts": 1, "dur": 2}]}).encode("utf-8")
    for bad in (good.replace(b"\\u00e9", b"\xc3"), good + b"\xff", b"\xef\xbb\xbf" + good,
                good.replace(b"\\u00e9", b"\xed\xa0\x80")):  # lone surrogate
        assert _ingest.parse_json(bad, False) == _ingest.UNSUPPORTED
    f = tmp_path / "t.json"
    f.write_bytes(good.replace(b"\\u00e9", b"\xc3"))
    with pytest.raises(MalformedTrace, match="not valid JSON"):
        parse_trace(f)


@pytest.mark.parametrize("special", ['\\"', "\\\\", "\\n", "\\u00e9", "\\ud83d\\ude00",
                                     "\x01", "\x1f", "\\x", "\\ud800", "é", "\x7f"])
def test_string_scan_around_16_byte_steps(special):
    """The string scanner steps 16 bytes at a time: an escape, a control
    character or the closing quote at every offset of a step (in a name, in
    a skipped value and in a key) reads like the Python reader or is
    declined where the reference errors."""
    for pos in range(0, 40):
        body = "a" * pos + special + "b" * (pos % 7)
        for rec in ('{"name": "%s", "ts": 1, "cat": "cpu_op"}' % body,
                    '{"name": "n", "ts": 1, "cat": "cpu_op", "x": "%s"}' % body,
                    '{"name": "n", "ts": 1, "cat": "cpu_op", "args": {"%s": 1}}' % body):
            check_text('{"traceEvents": [%s]}' % rec)
            check_text('[%s]' % rec)  # the closing quote near the end of the text
