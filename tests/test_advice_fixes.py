"""CPU: host-side edge behaviour that must match the reference.

* integral / fractional float request sizes replay like the reference's
  round_request (allocator.py:79-83), and a reused handle is DuplicateHandle
  before any size check (allocator.py:274-276);
* the config digest falls back to json for bools (json.dumps writes
  true/false, estimator.py:189-202);
* sequence numbers beyond the sequence-join key width are an engine limit,
  not a silent truncation.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import replay as oracle
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace
from paper_2504_03887_b200.errors import EngineLimitExceeded


def _oracle_peak(records):
    p = pack_trace(records)
    assert not p.host_errors
    offs = np.array([0, len(p.reqs)], dtype=np.int64)
    res, _ = oracle.replay_batch(p.reqs, offs, cfg_record(AllocatorConfig()))
    return int(res[0]["peak_allocated"]), int(res[0]["status"])


def test_float_sizes_pack_like_round_request():
    ints = [{"seq_no": 0, "kind": "alloc", "block_id": 1, "size": 1048576},
            {"seq_no": 1, "kind": "alloc", "block_id": 2, "size": 1025}]
    floats = [{"seq_no": 0, "kind": "alloc", "block_id": 1, "size": 1048576.0},
              {"seq_no": 1, "kind": "alloc", "block_id": 2, "size": 1024.25}]
    assert _oracle_peak(ints) == _oracle_peak(floats)
    p = pack_trace(floats)
    assert p.reqs["size"].tolist() == [1048576, 1025]
    # size in (0, 1) is positive for the reference: it rounds to one unit
    assert pack_trace([{"seq_no": 0, "kind": "alloc", "block_id": 1,
                        "size": 0.25}]).reqs["size"][0] == 1


def test_bad_size_on_reused_handle_is_duplicate_not_type_error():
    recs = [{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 512},
            {"seq_no": 1, "kind": "alloc", "block_id": "a", "size": "x"}]
    p = pack_trace(recs)
    assert not p.host_errors          # the kernel reports DuplicateHandle
    offs = np.array([0, 2], dtype=np.int64)
    res, _ = oracle.replay_batch(p.reqs, offs, cfg_record(AllocatorConfig()))
    assert int(res[0]["status"]) == 4 and int(res[0]["stop_index"]) == 1
    # a fresh handle with a bad size raises TypeError when reached
    p = pack_trace([{"seq_no": 0, "kind": "alloc", "block_id": "b", "size": "x"}])
    assert isinstance(p.host_errors[0], TypeError)


def test_digest_bool_params_fall_back_to_json():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.estimator import PeakMemoryEstimator
    bundle = synth_events.generate(leaves=20, iterations=2)
    for kw, cap, init in (({"iterations": True}, 0, 0),
                          ({}, False, 0), ({}, 0, True),
                          ({}, 1 << 64, 0)):
        est = PeakMemoryEstimator(**kw)
        assert est._digest(bundle, cap, init) == est._digest_json(bundle, cap, init)
    # and a bool would differ if it went through the native int writer
    est = PeakMemoryEstimator()
    assert est._digest_json(bundle, True, 0) != est._digest_json(bundle, 1, 0)


def test_sequence_numbers_beyond_32_bits_rejected():
    from paper_2504_03887_b200 import _pipeline
    with pytest.raises(EngineLimitExceeded):
        _pipeline.link([0], [1], [1 << 32], [], [], [], [0], [1])
    with pytest.raises(EngineLimitExceeded):
        _pipeline.link_roots([0], [1], [0, 1], [1 << 33], [0], [1], [], [])
