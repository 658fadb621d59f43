"""Parity-corpus helpers shared by the CPU (oracle) and GPU (engine) tests."""

from __future__ import annotations

import numpy as np

from oracle import sequencegen
from paper_2504_03887_b200.allocator import (AllocatorConfig, cfg_record,
                                             pack_trace)

CORPORA = {
    "corpus_seed1000": (1000, 1000, False),
    "corpus_seed2024": (2024, 300, False),
    "corpus_seed5eed": (0x5EED, 60, True),
}


def corpus(name: str):
    seed, count, cfg_first = CORPORA[name]
    gen = sequencegen.corpus_config_first if cfg_first else sequencegen.corpus
    return gen(seed, count)


def pack_corpus(cases):
    """Pack (sequence, params) pairs into one batch: (reqs, offsets, cfgs,
    cfg_of, packed)."""
    packed = [pack_trace(seq) for seq, _ in cases]
    cfgs = np.concatenate([
        cfg_record(AllocatorConfig(device_capacity=p["capacity"],
                                   max_split_size=p["max_split_size"]))
        for _, p in cases])
    offsets = np.zeros(len(cases) + 1, dtype=np.int64)
    np.cumsum([len(p.reqs) for p in packed], out=offsets[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    cfg_of = np.arange(len(cases), dtype=np.int32)
    return reqs, offsets, cfgs, cfg_of, packed


def timeline_rows(seq, tl, e0, n_ok):
    pairs = tl[2 * e0: 2 * (e0 + n_ok)].reshape(-1, 2).tolist()
    return [[r["seq_no"], a, b] for r, (a, b) in zip(seq, pairs)]


def compare_to_golden(cases, results, tl, offsets, gold_cases, digest):
    """Assert per-trace equality with the reference's golden values."""
    for i, ((seq, params), g) in enumerate(zip(cases, gold_cases)):
        r = results[i]
        ctx = f"case {i} params {params}"
        assert digest(seq) == g["sequence_sha256"], ctx
        assert int(r["peak_reserved"]) == g["peak_reserved"], ctx
        assert int(r["peak_allocated"]) == g["peak_allocated"], ctx
        assert int(r["final_reserved"]) == g["final_reserved"], ctx
        assert int(r["final_allocated"]) == g["final_allocated"], ctx
        assert int(r["n_segments_final"]) == g["n_segments_final"], ctx
        assert int(r["n_segments_peak"]) == g["n_segments_peak"], ctx
        assert int(r["max_free_blocks"]) == g["max_free_blocks"], ctx
        status = int(r["status"])
        if g["oom_seq_no"] is None:
            assert status == 0, ctx
            n_ok = len(seq)
        else:
            assert status == 1, ctx
            stop = int(r["stop_index"])
            assert seq[stop]["seq_no"] == g["oom_seq_no"], ctx
            n_ok = stop
        assert n_ok == g["timeline_len"], ctx
        rows = timeline_rows(seq, tl, int(offsets[i]), n_ok)
        assert digest(rows) == g["timeline_sha256"], ctx
