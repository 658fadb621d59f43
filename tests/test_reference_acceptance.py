"""The reference's acceptance cases (pkg/tests/test_acceptance.py) that sit
on the hot path, restated against this package: the segment-size table
(:70-87), 10k roundings (:90-97), the 1000-stream grouping property test
(:144-208), the fixture sequence invariants (:216-278) and the free-position
sensitivity case (:367-386)."""

from __future__ import annotations

import gzip
import math
import random
from collections import Counter

import pytest

from conftest import GOLDEN
from paper_2504_03887_b200.allocator import (AllocatorConfig, round_request,
                                             segment_size_for)
from paper_2504_03887_b200.trace import EventCategory, TraceEvent

MIB = 1 << 20
FIXTURES = ["tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"]


def test_segment_sizing_eight_point_table():
    table = {1: 2 * MIB, 512: 2 * MIB, MIB: 2 * MIB, MIB + 1: 20 * MIB,
             10 * MIB: 20 * MIB, 10 * MIB + 1: 12 * MIB, 11 * MIB: 12 * MIB,
             64 * MIB: 64 * MIB}
    cfg = AllocatorConfig()
    assert {s: segment_size_for(round_request(s), cfg) for s in table} == table


def test_rounding_on_10k_random_sizes():
    rng = random.Random(0xA11C)
    for _ in range(10_000):
        size = rng.randint(1, 64 * MIB)
        expected = 512 * ((size + 511) // 512)
        assert round_request(size) == expected == 512 * math.ceil(size / 512)


def _random_instant_stream(rng: random.Random):
    """Alloc/free instants over a small reused address pool plus the
    ground-truth pairing (test_acceptance.py:144-190, restated)."""
    events: list[TraceEvent] = []
    open_by_addr: dict[int, tuple[int, int]] = {}
    pairs: set[tuple[int, int, int]] = set()
    ts = 0
    pool = [0x1000 * (i + 1) for i in range(rng.randint(2, 8))]

    def emit(addr, nbytes):
        nonlocal ts
        ts += rng.randint(1, 3)
        events.append(TraceEvent(len(events), EventCategory.CPU_INSTANT_EVENT,
                                 "[memory]", ts, 0, addr=addr, nbytes=nbytes))

    for _ in range(rng.randint(1, 60)):
        roll = rng.random()
        closed = [a for a in pool if a not in open_by_addr]
        if (roll < 0.5 and closed) or not open_by_addr:
            if not closed:
                continue
            addr = rng.choice(closed)
            size = 512 * rng.randint(1, 64)
            emit(addr, size)
            open_by_addr[addr] = (events[-1].start_ts, size)
        elif roll < 0.9:
            addr = rng.choice(list(open_by_addr))
            alloc_ts, size = open_by_addr.pop(addr)
            emit(addr, -size)
            pairs.add((addr, alloc_ts, events[-1].start_ts))
        else:
            emit(0xDEAD000 + rng.randint(0, 3) * 0x10, -512)
    return events, pairs, {(a, t) for a, (t, _) in open_by_addr.items()}


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_grouping_pairs_frees_with_latest_open_alloc_1000_streams():
    from paper_2504_03887_b200.analysis import group_memory_events
    rng = random.Random(77)
    for case in range(1000):
        events, pairs, open_allocs = _random_instant_stream(rng)
        blocks = group_memory_events(events)
        assert len(blocks) == sum(1 for e in events if e.nbytes > 0), case
        assert {(b.addr, b.alloc_time, b.free_time) for b in blocks
                if b.free_time is not None} == pairs, case
        assert {(b.addr, b.alloc_time) for b in blocks
                if b.free_time is None} == open_allocs, case


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
@pytest.mark.parametrize("name", FIXTURES)
def test_training_sequence_invariants_on_fixtures(name, tmp_path):
    import paper_2504_03887_b200 as api
    trace = tmp_path / "trace.json"
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        trace.write_bytes(f.read())
    side = api.load_sidecar(GOLDEN / "traces" / f"{name}.sidecar.json")
    bundle = api.parse_trace(trace, sidecar=side)
    analyzed = api.analyze(bundle)
    seq = api.build_sequence(analyzed, iterations=2)
    reqs, tags, bounds = seq.requests, seq.phase_tags, seq.iteration_boundaries
    assert len(bounds) == 3
    A, F = api.RequestKind.ALLOC, api.RequestKind.FREE

    def role(r):
        return tags.get(r.block_id)

    model_bytes = sum(r.size for r in reqs if r.kind is A
                      and str(r.block_id).startswith("model:"))
    grad_bytes = sum(r.size for r in reqs if r.kind is A
                     and role(r) is api.BlockRole.GRADIENT
                     and bounds[0] <= r.virtual_ts < bounds[1])
    assert model_bytes == grad_bytes
    state = [r for r in reqs if r.kind is A
             and role(r) is api.BlockRole.OPTIMIZER_STATE]
    assert all(r.size in set(side.param_sizes) for r in state)
    resets = {m.start_ts for m in analyzed.markers
              if m.kind is api.MarkerKind.ZERO_GRAD}
    resets |= {t + bounds[-1] - bounds[-2] for t in resets}
    grad_frees = [r.virtual_ts for r in reqs
                  if r.kind is F and role(r) is api.BlockRole.GRADIENT]
    assert grad_frees and all(t in resets for t in grad_frees)

    def sizes(lo, hi):
        return Counter(r.size for r in reqs if r.kind is A
                       and lo <= r.virtual_ts < hi
                       and role(r) is not api.BlockRole.OPTIMIZER_STATE)
    assert sizes(bounds[0], bounds[1]) == sizes(bounds[1], bounds[2])
    if side.optimizer_name.lower() == "adam":
        assert sum(r.size for r in state) == 2 * sum(side.param_sizes)
        assert all(bounds[0] <= r.virtual_ts < bounds[1] for r in state)
    else:
        assert not state


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_peak_reserved_sensitive_to_free_position():
    import paper_2504_03887_b200 as api

    def alloc(s, b):
        return {"seq_no": s, "kind": "alloc", "block_id": b, "size": 15 * MIB,
                "stream": 0}

    def free(s, b):
        return {"seq_no": s, "kind": "free", "block_id": b, "size": 0, "stream": 0}

    overlapped = [alloc(0, "a"), alloc(1, "b"), free(2, "a"), free(3, "b")]
    serial = [alloc(0, "a"), free(1, "a"), alloc(2, "b"), free(3, "b")]
    p_over, p_ser = (r.peak_reserved for r in api.replay_batch([overlapped, serial]))
    assert p_over == 32 * MIB and p_ser == 16 * MIB
    assert (p_over - p_ser) / p_over >= 0.5
