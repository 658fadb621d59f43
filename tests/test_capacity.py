"""Batched capacity bisection (pm_capacity_search).

CPU: the oracle bisection (oracle/capacity.py) against the brute-force
definition -- the smallest runnable multiple of the segment-size unit --
on the reference-generated corpus and the GPT-2 capture sequences.
GPU: the engine's search against the oracle bisection, probe by probe
(capacity and the full replay result of every probe), bit-exact."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import capacity as ocap
from oracle import replay as oracle
from replay_cases import corpus, pack_corpus
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record

RESULT_FIELDS = ("peak_reserved", "peak_allocated", "final_reserved",
                 "final_allocated", "stop_index", "n_events_replayed", "status",
                 "n_segments_final", "n_segments_peak")


def c2():
    z = np.load(GOLDEN / "c2_sequences.npz")
    return z["reqs"], z["offsets"], json.loads(str(z["meta"]))


def corpus_batch(n=300):
    cases = corpus("corpus_seed1000")[:n]
    reqs, offsets, cfgs, cfg_of, _ = pack_corpus(cases)
    return reqs, offsets, cfgs, cfg_of


def test_oracle_bisection_matches_linear_scan_corpus():
    reqs, offsets, cfgs, cfg_of = corpus_batch(120)
    got = ocap.bisect(reqs, offsets, cfgs, cfg_of)
    checked = non_monotone = 0
    for t in range(len(offsets) - 1):
        if got["min_capacity"][t] < 0:
            continue
        want, monotone = ocap.linear_scan(reqs, offsets, cfgs[cfg_of[t]], t)
        if monotone:
            assert got["min_capacity"][t] == want, t
        else:
            non_monotone += 1
        checked += 1
    assert checked > 50
    assert non_monotone <= checked // 10


def test_oracle_bisection_matches_linear_scan_gpt2():
    reqs, offs, meta = c2()
    cfg = cfg_record(AllocatorConfig())
    got = ocap.bisect(reqs, offs, cfg)
    for t, m in enumerate(meta):
        assert got["unbounded"][t]["peak_reserved"] == m["peak_reserved"]
        want, monotone = ocap.linear_scan(reqs, offs, cfg[0], t)
        assert monotone, m["name"]
        assert got["min_capacity"][t] == want, m["name"]
        assert got["min_capacity"][t] <= m["peak_reserved"]


def test_bisection_bracket_invariants():
    """The answer runs and answer - unit OOMs (the bisection's contract)."""
    reqs, offsets, cfgs, cfg_of = corpus_batch(200)
    got = ocap.bisect(reqs, offsets, cfgs, cfg_of)
    for t in range(len(offsets) - 1):
        cap = got["min_capacity"][t]
        if cap <= 0:
            continue
        cfg = cfgs[cfg_of[t]].copy()
        sub = reqs[offsets[t]:offsets[t + 1]]
        for c, want in ((cap, 0), (cap - ocap._unit(cfg), 1)):
            cfg["device_capacity"] = c
            r, _ = oracle.replay_batch(sub, np.array([0, len(sub)]),
                                       np.array([cfg], dtype=oracle.CFG_DTYPE))
            assert int(r[0]["status"]) == want, (t, c)


def _compare(dev, want, n):
    assert list(dev["min_capacity"]) == list(want["min_capacity"])
    for t in range(n):
        for f in RESULT_FIELDS:
            assert dev["unbounded"][t][f] == want["unbounded"][t][f], (t, f)
        probes = want["probes"][t]
        assert int(dev["n_probes"][t]) == len(probes), t
        for k, (cap, r) in enumerate(probes):
            assert int(dev["probe_capacity"][k, t]) == cap, (t, k)
            for f in RESULT_FIELDS:
                assert dev["probe_results"][k, t][f] == r[f], (t, k, f)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_gpu_search_matches_oracle_corpus():
    from paper_2504_03887_b200.engine import DeviceBatch
    reqs, offsets, cfgs, cfg_of = corpus_batch(1000)
    dev = DeviceBatch(reqs, offsets, cfgs, cfg_of).capacity_search()
    _compare(dev, ocap.bisect(reqs, offsets, cfgs, cfg_of), len(offsets) - 1)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_gpu_search_matches_oracle_gpt2_and_c3():
    from paper_2504_03887_b200 import synth
    from paper_2504_03887_b200.engine import DeviceBatch
    reqs, offs, _ = c2()
    r3, o3 = synth.generate(48, first=4000)
    reqs = np.concatenate([reqs, r3])
    offs = np.concatenate([offs, o3[1:] + offs[-1]])
    for cfg in (AllocatorConfig(), AllocatorConfig(max_split_size=64 << 20),
                AllocatorConfig(k_large_buffer=32 << 20, k_round_large=4 << 20)):
        rec = cfg_record(cfg)
        dev = DeviceBatch(reqs, offs, rec).capacity_search()
        _compare(dev, ocap.bisect(reqs, offs, rec), len(offs) - 1)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_min_runnable_capacity_api():
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200.capacity import min_runnable_capacity
    seqs = [[{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 3 << 20},
             {"seq_no": 1, "kind": "alloc", "block_id": "b", "size": 300 << 10},
             {"seq_no": 2, "kind": "free", "block_id": "a", "size": 0},
             {"seq_no": 3, "kind": "alloc", "block_id": "c", "size": 12 << 20}],
            []]
    res = min_runnable_capacity(seqs)
    assert res[1].min_capacity == 0 and res[1].probes == []
    r = res[0]
    assert r.unbounded_peak == api.replay(seqs[0]).peak_reserved
    ok = api.replay(seqs[0], AllocatorConfig(device_capacity=r.min_capacity))
    assert ok.oom_seq_no is None
    bad = api.replay(seqs[0], AllocatorConfig(device_capacity=r.min_capacity - (2 << 20)))
    assert bad.oom_seq_no is not None
    for cap, oom in r.probes:
        assert api.replay(seqs[0], AllocatorConfig(device_capacity=cap)).oom_seq_no == oom
    with pytest.raises(api.MalformedSequence):
        min_runnable_capacity([[{"seq_no": 0, "kind": "free", "block_id": "x",
                                 "size": 0}]])
