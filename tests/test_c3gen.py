"""The C3 workload generator (workloads/c3gen.c) is SURVEY §8d's recipe:
trace i drawn from numpy.random.Generator(PCG64(1_000_003 + i)).  Pinned to
the numpy spec (oracle/c3gen.py) trace for trace, and the two compiled copies
(engine synth library, oracle library) agree."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import c3gen
from oracle import replay as oracle_replay


@pytest.fixture(scope="module")
def synth():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03887_b200 import synth as s
    return s


@pytest.mark.parametrize("seed", [0, 1, 5, 1_000_003, 1_010_002, 2**32 + 7, 2**63 + 11])
def test_pcg64_raw_matches_numpy(synth, seed):
    lib = synth._load()
    lib.pm_synth_pcg64_raw.argtypes = [ctypes.c_uint64, ctypes.c_int32,
                                       ctypes.c_void_p]
    out = np.zeros(64, dtype=np.uint64)
    lib.pm_synth_pcg64_raw(seed, 64, out.ctypes.data)
    assert (out == np.random.PCG64(seed).random_raw(64)).all()


@pytest.mark.parametrize("index", [0, 1, 2, 38, 777, 5000, 9999])
def test_trace_matches_numpy_spec(synth, index):
    reqs, offs = synth.generate_ids([index])
    spec = c3gen.trace(index)
    assert len(reqs) == len(spec)
    assert (reqs == spec).all()


def test_trace_shape():
    """10^5 +- 10 % requests, dense handles, every alloc freed at most once."""
    for index in (3, 4):
        t = c3gen.trace(index)
        assert 90_000 <= len(t) <= 125_000
        allocs = t["kind_stream"] == 0
        assert (t["handle"][allocs] == np.arange(allocs.sum())).all()
        freed = t["handle"][~allocs]
        assert len(np.unique(freed)) == len(freed)
        assert (t["size"][allocs] > 0).all()


def test_engine_and_oracle_generators_agree(synth):
    ids = np.array([9998, 12, 4000, 12], dtype=np.int32)
    a, oa = synth.generate_ids(ids)
    b, ob = oracle_replay.c3_traces(ids)
    assert (oa == ob).all() and (a == b).all()
