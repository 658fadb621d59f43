"""GPU: replay(validate=True) -- the validating build of the kernels checks
the allocator invariants of AllocatorState.check_invariants
(allocator.py:324-354; run after every allocate / free when validate=True,
:291-292 / :319-320) after EVERY request, on the engine's own state, and
raises AssertionError on a violation.

* the seed-1000 corpus (the reference's acceptance corpus, test_acceptance.py
  :105-124) and the seed-2024 invariants corpus (:127-136) replay clean and
  give the same results as the regular build, in the narrow main pass;
* the multi-stream / all-knob corpus replays clean through the wide tiers;
* C3 prefixes and a fragmenting trace replay clean in every retry pass;
* injected faults (pm_validate_inject) are caught at the request they hit.
"""

from __future__ import annotations

import numpy as np
import pytest

from config_goldens import check, multistream_batch
from conftest import golden
from oracle import c3gen
from paper_2504_03887_b200 import _native
from paper_2504_03887_b200.allocator import (AllocatorConfig, cfg_record,
                                             pack_trace, replay)
from replay_cases import compare_to_golden, corpus, pack_corpus
from conftest import digest

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]

MIB = 1 << 20


@pytest.fixture(autouse=True)
def no_injection():
    lib = _native.load_validate_library()
    lib.pm_validate_inject(0, 0)
    yield
    lib.pm_validate_inject(0, 0)


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("name", ["corpus_seed1000", "corpus_seed2024"])
def test_reference_corpora_replay_clean(name, packed, monkeypatch):
    """In the 12-warp CTAs the batch size selects, and packed into 24-warp
    CTAs (PM_SPREAD=0)."""
    if packed:
        monkeypatch.setenv("PM_SPREAD", "0")
    cases = corpus(name)
    reqs, offsets, cfgs, cfg_of, _ = pack_corpus(cases)
    res, tl = _native.replay_host(reqs, offsets, cfgs, cfg_of, True, validate=True)
    assert not (res["status"] == _native.PM_INVARIANT_VIOLATION).any()
    compare_to_golden(cases, res, tl, offsets,
                      golden(f"replay_{name}.json")["cases"], digest)
    plain, _ = _native.replay_host(reqs, offsets, cfgs, cfg_of, False)
    assert (plain == res).all()


def test_multistream_all_knobs_replay_clean():
    reqs, offs, cfgs, cfg_of, gold = multistream_batch()
    res, tl = _native.replay_host(reqs, offs, cfgs, cfg_of, True, validate=True)
    check(res, tl, offs, gold)


def test_c3_prefixes_and_retry_passes_clean():
    parts = [c3gen.trace(i)[:3000] for i in (11, 12, 13)]
    offs = np.zeros(4, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=offs[1:])
    reqs = np.concatenate(parts)
    cfg = cfg_record(AllocatorConfig())
    res, _ = _native.replay_host(reqs, offs, cfg, None, False, validate=True)
    want, _ = _native.replay_host(reqs, offs, cfg, None, False)
    assert (res == want).all()
    # a trace whose free blocks outgrow the main pass (> 32 buckets): 3000
    # 512 B blocks, every other one freed -- 1500 free blocks that never
    # coalesce -- then a few allocations that reuse them
    recs = [{"seq_no": i, "kind": "alloc", "block_id": i, "size": 512}
            for i in range(3000)]
    recs += [{"seq_no": 3000 + i, "kind": "free", "block_id": 2 * i}
             for i in range(1500)]
    recs += [{"seq_no": 4500 + i, "kind": "alloc", "block_id": 5000 + i,
              "size": 512} for i in range(40)]
    out = replay(recs, validate=True)
    assert out == replay(recs)
    p = pack_trace(recs)
    r, _ = _native.replay_host(p.reqs, np.array([0, len(p.reqs)]),
                               cfg_record(AllocatorConfig()), None, False,
                               validate=True)
    assert int(r[0]["max_free_blocks"]) >= 1500


def test_estimator_validate_on_fixture():
    import gzip
    from conftest import GOLDEN
    from paper_2504_03887_b200.estimator import PeakMemoryEstimator
    from paper_2504_03887_b200.trace import load_sidecar, parse_trace
    import tempfile, os
    name = "tiny_mlp_adam"
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.json")
        with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
            open(path, "wb").write(f.read())
        bundle = parse_trace(path, sidecar=load_sidecar(
            str(GOLDEN / "traces" / f"{name}.sidecar.json")))
    report = PeakMemoryEstimator(validate=True).estimate(bundle)
    assert report.canonical_json() == \
        golden("pipeline_golden.json")[name]["golden_report"]


@pytest.mark.parametrize("kind,invariant", [(1, 7), (2, 3)])
def test_injected_faults_are_caught(kind, invariant):
    lib = _native.load_validate_library()
    # narrow main pass (stream 0) and wide tier (stream 1)
    for stream in (0, 1):
        recs = [{"seq_no": i, "kind": "alloc", "block_id": i, "size": 512 * (i + 1),
                 "stream": stream} for i in range(12)]
        p = pack_trace(recs)
        offs = np.array([0, len(p.reqs)], dtype=np.int64)
        assert lib.pm_validate_inject(5, kind) == 0
        res, _ = _native.replay_host(p.reqs, offs, cfg_record(AllocatorConfig()),
                                     None, False, validate=True)
        assert int(res[0]["status"]) == _native.PM_INVARIANT_VIOLATION, stream
        assert int(res[0]["stop_index"]) == 5
        assert int(res[0]["max_free_blocks"]) == invariant
        with pytest.raises(AssertionError, match="invariant violated after request 5"):
            replay(recs, validate=True)
        lib.pm_validate_inject(0, 0)
    # the regular build has no injection hook
    assert _native.load_library().pm_validate_inject(5, 1) != 0
