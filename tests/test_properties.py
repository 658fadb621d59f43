"""Property-based tests (hypothesis), the counterparts of the reference's
test_allocator.py:42-44 (rounding up to 2^40) and :197-226 (simulator vs
oracle on generated sequences): generated sequences and configs through the
GPU engine (narrow main pass, retry passes, wide tiers as the case needs)
against the C oracle, full timelines."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_2504_03887_b200.allocator import (AllocatorConfig, cfg_record,
                                             pack_trace, round_request,
                                             segment_size_for)
from paper_2504_03887_b200.errors import ZeroSize

MIB = 1 << 20


@given(st.integers(min_value=1, max_value=1 << 40),
       st.sampled_from([1, 2, 512, 1024, 4096, 1 << 20]))
def test_round_request_properties(size, align):
    r = round_request(size, align)
    assert r % align == 0 and size <= r < size + align


@given(st.integers(max_value=0))
def test_round_request_rejects_non_positive(size):
    with pytest.raises(ZeroSize):
        round_request(size)


@given(st.integers(min_value=1, max_value=1 << 36))
def test_segment_size_table(size):
    # allocator.py:86-92 on the rounded size, default knobs
    r = round_request(size)
    seg = segment_size_for(r)
    if r <= MIB:
        assert seg == 2 * MIB
    elif r <= 10 * MIB:
        assert seg == 20 * MIB
    else:
        assert seg % (2 * MIB) == 0 and r <= seg < r + 2 * MIB


SIZES = st.one_of(st.integers(1, 4 * MIB), st.integers(1, 64 * MIB),
                  st.sampled_from([1, 511, 512, 513, MIB, MIB + 1, 10 * MIB,
                                   10 * MIB + 1, 20 * MIB, 100 * MIB]))


@st.composite
def sequences(draw):
    n = draw(st.integers(1, 120))
    live, seq, nxt = [], [], 0
    for _ in range(n):
        if live and draw(st.booleans()):
            bid = live.pop(draw(st.integers(0, len(live) - 1)))
            seq.append({"seq_no": len(seq), "kind": "free", "block_id": bid})
        else:
            stream = draw(st.sampled_from([0, 0, 0, 1]))
            seq.append({"seq_no": len(seq), "kind": "alloc", "block_id": nxt,
                        "size": draw(SIZES), "stream": stream})
            live.append(nxt)
            nxt += 1
    return seq


CONFIGS = st.builds(
    AllocatorConfig,
    max_split_size=st.sampled_from([None, 20 * MIB, 32 * MIB + 512, 64 * MIB]),
    alignment=st.sampled_from([512, 1024, 4096]),
    device_capacity=st.sampled_from([None, None, 24 * MIB, 64 * MIB, 200 * MIB]))


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
@settings(max_examples=60, deadline=None,
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
@given(st.lists(st.tuples(sequences(), CONFIGS), min_size=1, max_size=24))
def test_engine_equals_oracle_on_generated_batches(batch):
    from oracle import replay as oracle
    from paper_2504_03887_b200 import _native
    packed = [pack_trace(seq) for seq, _ in batch]
    offs = np.zeros(len(batch) + 1, dtype=np.int64)
    np.cumsum([len(p.reqs) for p in packed], out=offs[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    cfgs = np.concatenate([cfg_record(c) for _, c in batch])
    cof = np.arange(len(batch), dtype=np.int32)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfgs, cof, timeline=True)
    got, tl = _native.replay_host(reqs, offs, cfgs, cof, True)
    assert (got == want).all()
    assert (tl == tl_ref).all()
    words = _native.wire_pack(reqs, offs)
    if words is not None:
        got, tl = _native.replay_host_wire(words, offs, cfgs, cof, True)
        assert (got == want).all() and (tl == tl_ref).all()
