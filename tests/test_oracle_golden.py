"""CPU: pin the C oracle (oracle/replay_oracle.c) to the reference.

The golden vectors were produced by the reference implementation itself
(tests/golden/make_golden.py); the corpus is regenerated here by the
restated generator, whose output digests are part of the goldens.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import digest, golden
from oracle import replay as oracle
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace
from replay_cases import CORPORA, compare_to_golden, corpus, pack_corpus

MIB = 1 << 20


@pytest.mark.parametrize("name", sorted(CORPORA))
def test_oracle_matches_reference_corpus(name):
    cases = corpus(name)
    reqs, offsets, cfgs, cfg_of, _ = pack_corpus(cases)
    res, tl = oracle.replay_batch(reqs, offsets, cfgs, cfg_of, timeline=True)
    compare_to_golden(cases, res, tl, offsets,
                      golden(f"replay_{name}.json")["cases"], digest)


@pytest.mark.parametrize("fixture", ["tiny_mlp_sgd", "tiny_mlp_adam",
                                     "tiny_mlp_sgd_pregrad"])
def test_oracle_matches_reference_fixture_sequences(fixture):
    g = golden("replay_fixture_sequences.json")[fixture]
    p = pack_trace(g["records"])
    offs = np.array([0, len(p.reqs)], dtype=np.int64)
    res, tl = oracle.replay_batch(p.reqs, offs, cfg_record(AllocatorConfig()),
                                  timeline=True)
    r, want = res[0], g["result"]
    assert int(r["status"]) == 0
    for k in ("peak_reserved", "peak_allocated", "final_reserved",
              "final_allocated", "n_segments_final", "n_segments_peak",
              "max_free_blocks"):
        assert int(r[k]) == want[k], k
    rows = [[rec["seq_no"], int(a), int(b)] for rec, (a, b) in
            zip(g["records"], tl.reshape(-1, 2))]
    assert rows == want["timeline"]


def _one(reqs, cfg=None):
    p = pack_trace(reqs)
    offs = np.array([0, len(p.reqs)], dtype=np.int64)
    res, tl = oracle.replay_batch(p.reqs, offs, cfg_record(cfg or AllocatorConfig()),
                                  timeline=True)
    return res[0], tl


def test_oracle_hand_scenarios():
    # test_reference_allocator.py:141-151 -- release then fit
    r, _ = _one([{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 11 * MIB},
                 {"seq_no": 1, "kind": "free", "block_id": "a"},
                 {"seq_no": 2, "kind": "alloc", "block_id": "b", "size": 15 * MIB}],
                AllocatorConfig(device_capacity=22 * MIB))
    assert int(r["final_reserved"]) == 16 * MIB
    assert int(r["peak_reserved"]) == 16 * MIB
    # test_reference_allocator.py:160-175 -- over-threshold first
    r, _ = _one([{"seq_no": 0, "kind": "alloc", "block_id": "big", "size": 30 * MIB},
                 {"seq_no": 1, "kind": "alloc", "block_id": "small", "size": 512},
                 {"seq_no": 2, "kind": "free", "block_id": "big"},
                 {"seq_no": 3, "kind": "free", "block_id": "small"},
                 {"seq_no": 4, "kind": "alloc", "block_id": "mid", "size": 5 * MIB}],
                AllocatorConfig(device_capacity=34 * MIB, max_split_size=20 * MIB))
    assert int(r["final_reserved"]) == 22 * MIB
    assert int(r["n_segments_final"]) == 2
    # releases are not undone by an OOM
    r, _ = _one([{"seq_no": 0, "kind": "alloc", "block_id": 1, "size": 512},
                 {"seq_no": 1, "kind": "free", "block_id": 1},
                 {"seq_no": 2, "kind": "alloc", "block_id": 2, "size": 30 * MIB}],
                AllocatorConfig(device_capacity=20 * MIB))
    assert int(r["status"]) == 1 and int(r["stop_index"]) == 2
    assert int(r["final_reserved"]) == 0 and int(r["peak_reserved"]) == 2 * MIB
