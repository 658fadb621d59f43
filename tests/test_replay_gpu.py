"""GPU parity: the batched replay kernel vs the reference (golden vectors)
and vs the C oracle, through the C ABI and the reference-mirroring API.

Reference behaviour pinned here: allocator.py:155-393 (replay), the
hand-computed scenarios of test_reference_allocator.py / test_allocator.py,
the 1000-case seed-1000 equivalence corpus (test_acceptance.py:105-124) and
the committed fixtures' orchestrated sequences.
"""

from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import digest, golden
from oracle import replay as oracle
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import (AllocatorConfig, cfg_record,
                                             pack_trace, replay, replay_batch)
from paper_2504_03887_b200.engine import DeviceBatch
from paper_2504_03887_b200.errors import MalformedSequence, ZeroSize
from replay_cases import CORPORA, compare_to_golden, corpus, pack_corpus

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]

MIB = 1 << 20


def alloc(seq, bid, size, **kw):
    return {"seq_no": seq, "kind": "alloc", "block_id": bid, "size": size, **kw}


def free(seq, bid):
    return {"seq_no": seq, "kind": "free", "block_id": bid}


def assert_same(got, want):
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} traces differ, first {bad[:5]}: " \
        f"{got[bad[0]]} vs {want[bad[0]]}"


# --- golden corpora (reference-generated) -----------------------------------

@pytest.mark.parametrize("width", ["auto", "packed", "one_warp", "n2000", "n2600"])
@pytest.mark.parametrize("name", sorted(CORPORA))
def test_engine_matches_reference_corpus(name, width, monkeypatch):
    """Every main-pass width on the corpus: the batch as it comes (the
    narrowest CTA that holds it: 12 warps for a corpus), the packed 24-warp
    CTAs (PM_SPREAD=0), batches of at most one trace per SM (one warp per
    CTA), and the corpus repeated to 2000 / 2600 traces (16 / 20 warps per
    CTA on 148 SMs)."""
    cases = corpus(name)
    want = golden(f"replay_{name}.json")["cases"]
    if width == "packed":
        monkeypatch.setenv("PM_SPREAD", "0")
    if width.startswith("n"):
        m = int(width[1:])
        k = -(-m // len(cases))
        cases, want = (cases * k)[:m], (want * k)[:m]
    step = 100 if width == "one_warp" else len(cases)
    for a in range(0, len(cases), step):
        part = cases[a:a + step]
        reqs, offsets, cfgs, cfg_of, _ = pack_corpus(part)
        res, tl = _native.replay_host(reqs, offsets, cfgs, cfg_of, True)
        compare_to_golden(part, res, tl, offsets, want[a:a + step], digest)


@pytest.mark.parametrize("fixture", ["tiny_mlp_sgd", "tiny_mlp_adam",
                                     "tiny_mlp_sgd_pregrad"])
def test_engine_matches_reference_fixture_sequences(fixture):
    g = golden("replay_fixture_sequences.json")[fixture]
    out = replay(g["records"])
    want = g["result"]
    assert out.peak_reserved == want["peak_reserved"]
    assert out.peak_allocated == want["peak_allocated"]
    assert out.final_reserved == want["final_reserved"]
    assert out.final_allocated == want["final_allocated"]
    assert out.n_segments_final == want["n_segments_final"]
    assert out.n_segments_peak == want["n_segments_peak"]
    assert [list(t) for t in out.timeline] == want["timeline"]
    assert out.oom_seq_no is None


# --- hand-computed scenarios (test_reference_allocator.py, test_allocator.py)

def test_alloc_free_timeline():
    out = replay([alloc(0, 1, 512), free(1, 1)])
    assert out.peak_reserved == 2 * MIB and out.peak_allocated == 512
    assert out.timeline == [(0, 2 * MIB, 512), (1, 2 * MIB, 0)]
    assert out.oom_seq_no is None


def test_empty_sequence():
    out = replay([])
    assert (out.peak_reserved, out.peak_allocated, out.timeline) == (0, 0, [])


def test_second_alloc_reuses_remainder():
    out = replay([alloc(0, "h1", 512), alloc(1, "h2", 512)])
    assert out.timeline[-1] == (1, 2 * MIB, 1024)
    assert out.n_segments_final == 1


def test_best_fit_prefers_smallest_hole():
    # holes of 1024 (offset 0) and 512 (offset 5120); e must take the 512 one:
    # freeing e afterwards then re-allocating 1024 must reuse offset 0 whole
    seq = [alloc(0, "a", 1024), alloc(1, "b", 4096), alloc(2, "c", 512),
           alloc(3, "d", 4096), free(4, "a"), free(5, "c"), alloc(6, "e", 512)]
    out = replay(seq)
    assert out.timeline[-1] == (6, 2 * MIB, 4096 + 512 + 4096)
    p = pack_trace(seq)
    res, _ = oracle.replay_batch(p.reqs, np.array([0, len(seq)]),
                                 cfg_record(AllocatorConfig()))
    assert res[0]["max_free_blocks"] == 3


def test_coalesce_both_sides():
    seq = [alloc(0, "A", 1024), alloc(1, "B", 1024), alloc(2, "C", 1024),
           free(3, "A"), free(4, "C"), free(5, "B"),
           alloc(6, "D", 2 * MIB)]  # fits only if the segment is whole again
    out = replay(seq)
    assert out.timeline[-1] == (6, 2 * MIB, 2 * MIB)
    assert out.n_segments_peak == 1


def test_release_then_fit():
    out = replay([alloc(0, "a", 11 * MIB), free(1, "a"), alloc(2, "b", 15 * MIB)],
                 AllocatorConfig(device_capacity=22 * MIB))
    assert out.final_reserved == 16 * MIB and out.peak_reserved == 16 * MIB
    assert out.final_allocated == 15 * MIB


def test_partially_used_segment_never_released():
    out = replay([alloc(0, "a", 512), alloc(1, "b", 2 * MIB)],
                 AllocatorConfig(device_capacity=4 * MIB))
    assert out.oom_seq_no == 1 and out.final_reserved == 2 * MIB


def test_over_threshold_released_first_largest_first():
    t = 20 * MIB
    out = replay([alloc(0, "big", 30 * MIB), alloc(1, "small", 512),
                  free(2, "big"), free(3, "small"), alloc(4, "mid", 5 * MIB)],
                 AllocatorConfig(device_capacity=34 * MIB, max_split_size=t))
    assert out.timeline[3] == (3, 32 * MIB, 0)
    assert out.final_reserved == 22 * MIB and out.n_segments_final == 2


def test_oversize_block_handed_out_whole():
    cfg = AllocatorConfig(max_split_size=20 * MIB)
    out = replay([alloc(0, "a", 30 * MIB), free(1, "a"), alloc(2, "b", 25 * MIB)], cfg)
    assert out.final_reserved == 30 * MIB and out.final_allocated == 30 * MIB


def test_small_request_skips_oversize_block():
    cfg = AllocatorConfig(max_split_size=20 * MIB)
    out = replay([alloc(0, "a", 30 * MIB), free(1, "a"), alloc(2, "b", MIB)], cfg)
    assert out.final_reserved == 32 * MIB and out.final_allocated == MIB


def test_oom_is_a_verdict_and_releases_stick():
    out = replay([alloc(0, 1, 512), alloc(1, 2, 5 * MIB)],
                 AllocatorConfig(device_capacity=3 * MIB))
    assert out.oom_seq_no == 1 and out.timeline == [(0, 2 * MIB, 512)]
    out = replay([alloc(0, 1, 512), free(1, 1), alloc(2, 2, 30 * MIB)],
                 AllocatorConfig(device_capacity=20 * MIB))
    assert out.oom_seq_no == 2 and out.final_reserved == 0
    assert out.peak_reserved == 2 * MIB


def test_budget_zero_ooms_first_alloc():
    out = replay([alloc(0, 1, 512)], AllocatorConfig(device_capacity=0))
    assert out.oom_seq_no == 0 and out.timeline == []


def test_free_position_changes_peak():
    hold = [alloc(0, 1, 15 * MIB), alloc(1, 2, 15 * MIB), free(2, 1), free(3, 2)]
    eager = [alloc(0, 1, 15 * MIB), free(1, 1), alloc(2, 2, 15 * MIB), free(3, 2)]
    assert replay(hold).peak_reserved == 32 * MIB
    assert replay(eager).peak_reserved == 16 * MIB


def test_seq_no_is_copied_not_indexed():
    out = replay([alloc(70, "x", 512), free(5, "x")])
    assert [t[0] for t in out.timeline] == [70, 5]


# --- error precedence (allocator.py:371-385) --------------------------------

def test_free_before_alloc_is_malformed():
    with pytest.raises(MalformedSequence):
        replay([free(0, 7)])


def test_double_free_is_malformed():
    with pytest.raises(MalformedSequence):
        replay([alloc(0, 1, 512), free(1, 1), free(2, 1)])


def test_duplicate_handle_even_after_free():
    with pytest.raises(MalformedSequence):
        replay([alloc(0, "h", 512), free(1, "h"), alloc(2, "h", 512)])


def test_zero_size_unwrapped():
    with pytest.raises(ZeroSize):
        replay([alloc(0, 1, 0)])


def test_duplicate_checked_before_zero_size():
    with pytest.raises(MalformedSequence):
        replay([alloc(0, 1, 512), alloc(1, 1, 0)])


def test_unknown_kind():
    with pytest.raises(MalformedSequence):
        replay([{"seq_no": 0, "kind": "resize", "block_id": 1}])


def test_missing_size_is_keyerror():
    with pytest.raises(KeyError):
        replay([{"seq_no": 0, "kind": "alloc", "block_id": 1}])


def test_oom_shadows_later_errors():
    # replay stops at the OOM; the malformed request after it is never read
    out = replay([alloc(0, 1, 512), alloc(1, 2, 30 * MIB), free(2, 99),
                  {"seq_no": 3, "kind": "alloc", "block_id": 5}],
                 AllocatorConfig(device_capacity=4 * MIB))
    assert out.oom_seq_no == 1


# --- engine vs oracle on wider inputs ----------------------------------------

def _random_multistream(rng, n):
    live, seq, nxt = [], [], 0
    for _ in range(n):
        if live and rng.random() < 0.45:
            bid = live.pop(rng.randrange(len(live)))
            seq.append(free(len(seq), bid))
        else:
            size = rng.choice([rng.randint(1, 4 * MIB), rng.randint(1, 64 * MIB),
                               rng.choice([512, MIB, 10 * MIB + 1, 20 * MIB])])
            seq.append(alloc(len(seq), nxt, size, stream=rng.choice([0, 0, 1, 3])))
            live.append(nxt)
            nxt += 1
    return seq


def test_multistream_and_configs_vs_oracle():
    rng = random.Random(4242)
    traces, cfgs = [], []
    grid = [AllocatorConfig(max_split_size=ms, alignment=al, **seg,
                            device_capacity=cap)
            for ms in (None, 20 * MIB, 64 * MIB)
            for al in (512, 4096)
            for seg in ({}, {"k_small_buffer": 4 * MIB}, {"k_round_large": 4 * MIB})
            for cap in (None, 96 * MIB)]
    for cfg in grid:
        for _ in range(6):
            traces.append(_random_multistream(rng, rng.randint(50, 600)))
            cfgs.append(cfg)
    packed = [pack_trace(t) for t in traces]
    offs = np.zeros(len(traces) + 1, dtype=np.int64)
    np.cumsum([len(p.reqs) for p in packed], out=offs[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    carr = np.concatenate([cfg_record(c) for c in cfgs])
    cof = np.arange(len(traces), dtype=np.int32)
    got, tl = _native.replay_host(reqs, offs, carr, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, carr, cof, timeline=True)
    assert_same(got, want)
    assert (tl == tl_ref).all()


def test_pool_overflow_retry_path_vs_oracle():
    # > pool capacity non-adjacent free blocks: allocate 3000 blocks of 512 B,
    # free every other one -> 1500 separate holes, then allocate into them
    seq = [alloc(i, i, 512) for i in range(3000)]
    seq += [free(3000 + k, 2 * k) for k in range(1500)]
    seq += [alloc(4500 + k, 10_000 + k, 512) for k in range(700)]
    p = pack_trace(seq)
    offs = np.array([0, len(seq)], dtype=np.int64)
    got, tl = _native.replay_host(p.reqs, offs, cfg_record(AllocatorConfig()),
                                  None, True)
    want, tl_ref = oracle.replay_batch(p.reqs, offs, cfg_record(AllocatorConfig()),
                                       timeline=True)
    assert int(want[0]["max_free_blocks"]) > 1024
    assert_same(got, want)
    assert (tl == tl_ref).all()


def test_synthetic_llama_traces_vs_oracle():
    reqs, offs = synth.generate(24)
    cfgs = np.concatenate([cfg_record(AllocatorConfig()),
                           cfg_record(AllocatorConfig(max_split_size=64 * MIB)),
                           cfg_record(AllocatorConfig(device_capacity=64 << 30))])
    cof = (np.arange(24) % 3).astype(np.int32)
    got, tl = _native.replay_host(reqs, offs, cfgs, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfgs, cof, timeline=True)
    assert_same(got, want)
    assert (tl == tl_ref).all()


def test_device_batch_repeatable_and_matches_host_path():
    reqs, offs = synth.generate(40, first=100)
    cfg = cfg_record(AllocatorConfig())
    batch = DeviceBatch(reqs, offs, cfg)
    batch.launch()
    first = batch.results()
    batch.launch()
    second = batch.results()
    assert_same(first, second)
    want, _ = oracle.replay_batch(reqs, offs, cfg)
    assert_same(first, want)


def test_replay_batch_api():
    rng = random.Random(9)
    traces = [_random_multistream(rng, 200) for _ in range(10)]
    outs = replay_batch(traces, [AllocatorConfig(device_capacity=64 * MIB)] * 10)
    for t, o in zip(traces, outs):
        single = replay(t, AllocatorConfig(device_capacity=64 * MIB))
        assert o.timeline == single.timeline and o.oom_seq_no == single.oom_seq_no


def test_many_traces_per_warp_vs_oracle(monkeypatch):
    # persistent warps replay trace after trace: cap the grid so every warp
    # handles several traces (state must not leak between them)
    monkeypatch.setenv("PM_MAX_GRID", "3")
    reqs, offs = synth.generate(12, first=500)
    cfg = cfg_record(AllocatorConfig())
    got, tl = _native.replay_host(reqs, offs, cfg, None, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert_same(got, want)
    assert (tl == tl_ref).all()
    cases = corpus("corpus_seed1000")[:300]
    r2, o2, c2, f2, _ = pack_corpus(cases)
    got, tl = _native.replay_host(r2, o2, c2, f2, True)
    want, tl_ref = oracle.replay_batch(r2, o2, c2, f2, timeline=True)
    assert_same(got, want)
    assert (tl == tl_ref).all()


def test_hbm_tier_vs_oracle():
    # 10k non-adjacent free blocks outgrow the shared-memory tiers (~9k
    # entries) and land in tier 3 (shared-memory directory, HBM entries)
    seq = [alloc(i, i, 512) for i in range(20_000)]
    seq += [free(20_000 + k, 2 * k) for k in range(10_000)]
    seq += [alloc(30_000 + k, 50_000 + k, 512) for k in range(3_000)]
    p = pack_trace(seq)
    offs = np.array([0, len(seq)], dtype=np.int64)
    got, tl = _native.replay_host(p.reqs, offs, cfg_record(AllocatorConfig()),
                                  None, True)
    want, tl_ref = oracle.replay_batch(p.reqs, offs, cfg_record(AllocatorConfig()),
                                       timeline=True)
    assert int(want[0]["max_free_blocks"]) >= 10_000
    assert_same(got, want)
    assert (tl == tl_ref).all()


def _holes(n_holes, fill):
    seq = [alloc(i, i, 512) for i in range(2 * n_holes)]
    seq += [free(2 * n_holes + k, 2 * k) for k in range(n_holes)]
    seq += [alloc(3 * n_holes + k, 10 * n_holes + k, 512) for k in range(fill)]
    return seq


def test_retry_passes_vs_oracle():
    # 2k holes outgrow the main pass's 32-bucket register directory and
    # finish in pass 1 (shared-memory directory and entries); 20k outgrow
    # its ~430 buckets and finish in pass 2 (HBM entries); 400k outgrow pass
    # 2's ~9.6k-bucket directory and finish in wide tier 4
    traces = [_holes(2_000, 500), _holes(20_000, 2_000), _holes(400_000, 3_000)]
    packed = [pack_trace(t) for t in traces]
    offs = np.zeros(4, dtype=np.int64)
    np.cumsum([len(p.reqs) for p in packed], out=offs[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    cfg = cfg_record(AllocatorConfig())
    batch = DeviceBatch(reqs, offs, cfg)
    batch.launch()
    got = batch.results()
    passes = batch.tier_counts()
    want, _ = oracle.replay_batch(reqs, offs, cfg)
    assert_same(got, want)
    assert int(want[2]["max_free_blocks"]) >= 400_000
    # narrow passes 1 (multi-warp shared-memory pools), 2 (one warp per SM),
    # 3 (HBM entries), then wide tier 4 for the 400k-free-block trace
    assert passes[0] == 3 and passes[1] >= 2 and passes[2] >= 1, passes
    assert passes[6] == 1, passes
