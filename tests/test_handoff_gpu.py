"""GPU: traces that outgrow a pass continue in the next one from a
checkpoint (csrc/replay_narrow.cuh NCk) instead of replaying again from
request 0 -- results and FULL timelines equal the oracle's whichever pass
finishes a trace, for pm_req_t and wire-word input, including traces handed
on twice (pass 1 -> 2 -> 3) and the validating build (invariants checked
after every request, before and after each resume)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import replay as oracle
from paper_2504_03887_b200 import _native
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace
from paper_2504_03887_b200.engine import DeviceBatch

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def _fragmented(n_traces=12, leaves=10000):
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    parts = []
    for v in range(n_traces):
        b = synth_events.generate(leaves + 53 * v, 2, seed=100 + v)
        parts.append(api.build_sequence(api.analyze(b), 2).packed)
    offs = np.zeros(len(parts) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=offs[1:])
    return np.concatenate(parts), offs


def _holes(n_blocks, keep_every):
    """n_blocks 512 B blocks, all but every keep_every-th freed: n_blocks free
    blocks that never coalesce (a free-block count that grows steadily)."""
    recs = [{"seq_no": i, "kind": "alloc", "block_id": i, "size": 512}
            for i in range(n_blocks)]
    recs += [{"seq_no": n_blocks + k, "kind": "free", "block_id": i}
             for k, i in enumerate(i for i in range(n_blocks) if i % 2 == 0)]
    return pack_trace(recs).reqs


@pytest.fixture(scope="module")
def frag():
    return _fragmented()


def test_fragmented_traces_resume_in_pass1_device(frag):
    reqs, offs = frag
    cfg = cfg_record(AllocatorConfig())
    b = DeviceBatch(reqs, offs, cfg, timeline=True)
    b.launch()
    got, tl = b.results(), b.timeline()
    passes = b.tier_counts()
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert (got == want).all()
    assert (tl == tl_ref[:len(tl)]).all()
    assert passes[0] == len(offs) - 1, passes  # every trace was handed off
    assert int(want["max_free_blocks"].min()) > 1024


def test_fragmented_traces_resume_wire_host(frag):
    reqs, offs = frag
    reqs = reqs.copy()
    # the wire format numbers handles by allocation order: renumber
    for t in range(len(offs) - 1):
        r = reqs[offs[t]:offs[t + 1]]
        alloc = (r["kind_stream"] & 3) == 0
        new = np.full(len(r), -1, dtype=np.int64)
        new[r["handle"][alloc]] = np.arange(int(alloc.sum()))
        r["handle"] = new[r["handle"]]
    cfg = cfg_record(AllocatorConfig())
    words = _native.wire_pack(reqs, offs)
    assert words is not None
    got, tl = _native.replay_host_wire(words, offs, cfg, None, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert (got == want).all()
    assert (tl == tl_ref).all()


def test_handed_on_twice_and_validated():
    # free-block counts of ~3k (outgrows pass 1's pools), ~20k (outgrows
    # pass 2's), ~60k (pass 3): each continues from its last checkpoint
    parts = [_holes(6_000, 2), _holes(40_000, 2), _holes(120_000, 2)]
    offs = np.zeros(4, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=offs[1:])
    reqs = np.concatenate(parts)
    cfg = cfg_record(AllocatorConfig())
    b = DeviceBatch(reqs, offs, cfg, timeline=True)
    b.launch()
    got, tl = b.results(), b.timeline()
    passes = b.tier_counts()
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert (got == want).all()
    assert (tl == tl_ref[:len(tl)]).all()
    assert passes[0] == 3 and passes[1] >= 2 and passes[2] >= 1, passes
    # the validating build on the two smaller ones (O(state) per request)
    k = int(offs[2])
    res, tlv = _native.replay_host(reqs[:k], offs[:3], cfg, None, True, validate=True)
    assert (res == want[:2]).all()
    assert (tlv == tl_ref[:2 * k]).all()


def test_c5_size_trace_vs_oracle():
    """BASELINE's C5 at its stated size: one 10^7-event trace (357,200 leaf
    layers, 2 iterations -> 4.29 M requests, 45 k free blocks at peak) --
    main pass, pass 1, pass 1b, then pass 2, whose directory is kept under
    its soft size by merging -- equals the oracle, full timeline included."""
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    b = synth_events.generate(357_200, 2)
    assert len(b.start) > 10_000_000
    reqs = api.build_sequence(api.analyze(b), 2).packed
    offs = np.array([0, len(reqs)], dtype=np.int64)
    cfg = cfg_record(AllocatorConfig())
    d = DeviceBatch(reqs, offs, cfg, timeline=True)
    d.launch()
    got, tl = d.results(), d.timeline()
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert (got == want).all()
    assert (tl == tl_ref[:len(tl)]).all()
    assert int(want["max_free_blocks"][0]) > 40_000
    assert d.tier_counts()[2] == 1  # finished in pass 2
