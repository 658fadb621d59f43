"""Batches and checks for the configuration goldens produced by the
reference itself (tests/golden/make_golden_configs.py): the C4 config grid,
multi-stream sequences over all eight allocator knobs, and full C3 traces.
Shared by the oracle (CPU) and engine (GPU) tests."""

from __future__ import annotations

import hashlib
import json

import numpy as np

from c4_cases import c4_batch, c4_configs, timeline_digest
from conftest import GOLDEN, golden
from oracle import c3gen, sequencegen
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace

FIELDS = ("peak_reserved", "peak_allocated", "final_reserved", "final_allocated",
          "n_segments_final", "n_segments_peak", "max_free_blocks")


def _sha(reqs) -> str:
    return hashlib.sha256(np.ascontiguousarray(reqs).tobytes()).hexdigest()


def c4_grid_batch():
    """(reqs, offsets, cfg records, cfg_of, gold results), replica-major as
    the golden file: replica t * 69 + c = trace t under grid config c."""
    g = golden("replay_c4_grid.json")
    z = np.load(GOLDEN / "c2_sequences.npz", allow_pickle=True)
    parts = []
    for t in g["traces"]:
        if t["source"] == "c3":
            r = c3gen.trace(t["index"])[:t["n_requests"]]
        else:
            k = t["index"]
            r = z["reqs"][z["offsets"][k]:z["offsets"][k + 1]]
        assert _sha(r) == t["sequence_sha256"], t["name"]
        parts.append(r)
    offs = np.zeros(len(parts) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=offs[1:])
    reqs = np.concatenate(parts)
    cfgs = c4_configs()
    assert len(cfgs) == len(g["configs"])
    big, boffs, rec, cfg_of = c4_batch(reqs, offs, cfgs)
    return big, boffs, rec, cfg_of, g["results"]


def multistream_batch():
    g = golden("replay_multistream.json")
    cases = sequencegen.multistream_corpus(g["seed"], g["count"])
    packed, cfgs = [], []
    for (seq, cfg), gc in zip(cases, g["cases"]):
        assert hashlib.sha256(json.dumps(seq, sort_keys=True, separators=(
            ",", ":")).encode()).hexdigest() == gc["sequence_sha256"]
        packed.append(pack_trace(seq).reqs)
        cfgs.append(cfg_record(AllocatorConfig(**cfg)))
    offs = np.zeros(len(packed) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in packed], out=offs[1:])
    cfg_of = np.arange(len(packed), dtype=np.int32)
    return np.concatenate(packed), offs, np.concatenate(cfgs), cfg_of, g["cases"]


def c3_full_batch(generate):
    """`generate(ids) -> (reqs, offsets)`: the engine's synth library or the
    oracle library's copy of the generator."""
    g = golden("replay_c3_full.json")
    reqs, offs = generate(np.array(g["ids"], dtype=np.int32))
    for k, gc in enumerate(g["cases"]):
        assert _sha(reqs[offs[k]:offs[k + 1]]) == gc["sequence_sha256"], gc["trace"]
    cfg = cfg_record(AllocatorConfig())
    return reqs, offs, cfg, None, g["cases"]


def check(results, tl, offs, gold) -> int:
    """Every field + the timeline digest of every case; returns cases."""
    assert len(results) == len(gold)
    for i, g in enumerate(gold):
        r = results[i]
        for f in FIELDS:
            assert int(r[f]) == g[f], (i, f, int(r[f]), g[f])
        status = int(r["status"])
        if g["error"] is not None:
            raise AssertionError(f"golden case {i} ends in {g['error']}")
        if g["oom_seq_no"] is None:
            assert status == 0, (i, status)
            n_ok = int(offs[i + 1] - offs[i])
        else:
            assert status == 1, (i, status)
            n_ok = int(r["stop_index"])
            assert n_ok == g["oom_seq_no"], i      # seq_no == index here
        assert n_ok == g["timeline_len"], i
        if tl is not None:
            pairs = tl[2 * int(offs[i]): 2 * (int(offs[i]) + n_ok)]
            assert timeline_digest(pairs) == g["timeline_sha256"], i
    return len(gold)
