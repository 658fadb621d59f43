"""CPU: the C-ABI library builds, loads and exports what the header declares;
host-side packing mirrors the reference's per-request reads."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import REPO
from paper_2504_03887_b200 import _native
from paper_2504_03887_b200.allocator import (AllocatorConfig, pack_trace,
                                             round_request, segment_size_for)
from paper_2504_03887_b200.errors import ZeroSize

MIB = 1 << 20
HEADER = REPO / "include" / "peakmem_b200.h"
PIPE_HEADER = REPO / "include" / "peakmem_pipeline.h"


def header_functions(header=HEADER):
    text = header.read_text()
    return sorted(set(re.findall(
        r"^\s*(?:int|int64_t|void|const char\*)\s+(pm_\w+)\(",
        text, re.M)))


def test_header_declares_what_python_binds():
    assert header_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.LIB_PATH
    if not lib.exists():
        import __graft_entry__
        __graft_entry__.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pm_\w+)", out))
    for sym in header_functions():
        assert sym in exported, sym
    loaded = _native.load_library()
    assert loaded.pm_version() == 2


def test_pipeline_library_exports_every_declared_symbol():
    from paper_2504_03887_b200 import _pipeline
    assert header_functions(PIPE_HEADER) == sorted(_pipeline.EXPORTED_SYMBOLS)
    lib = _pipeline.LIB_PATH
    if not lib.exists():
        import __graft_entry__
        __graft_entry__.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pm_\w+)", out))
    for sym in header_functions(PIPE_HEADER):
        assert sym in exported, sym
    _pipeline.load()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_sizing_is_host_only():
    small = _native.workspace_bytes(1000, 100, 10)
    big = _native.workspace_bytes(10_000, 100, 10)
    assert big - small >= 16 * 9000 - 256  # 16 B record per request


def test_struct_layouts_match_header():
    assert _native.REQ_DTYPE.itemsize == 16
    assert _native.CFG_DTYPE.itemsize == 64
    assert _native.RESULT_DTYPE.itemsize == 64


# --- host-side arithmetic and packing (reference: allocator.py:49-92) -----

@pytest.mark.parametrize("size,expected", [(1, 512), (512, 512), (513, 1024),
                                           (511, 512), (1024, 1024), (4097, 4608)])
def test_round_request(size, expected):
    assert round_request(size) == expected


def test_round_request_zero():
    with pytest.raises(ZeroSize):
        round_request(0)


def test_segment_table():
    table = {1: 2 * MIB, 512: 2 * MIB, MIB: 2 * MIB, MIB + 1: 20 * MIB,
             10 * MIB: 20 * MIB, 10 * MIB + 1: 12 * MIB, 11 * MIB: 12 * MIB,
             64 * MIB: 64 * MIB}
    cfg = AllocatorConfig()
    assert {s: segment_size_for(round_request(s), cfg) for s in table} == table


def test_config_validation():
    with pytest.raises(ValueError):
        AllocatorConfig(alignment=500)
    with pytest.raises(ValueError):
        AllocatorConfig(max_split_size=8 * MIB)
    assert AllocatorConfig(max_split_size=20 * MIB).max_split_size == 20 * MIB


def test_pack_interns_ids_and_streams():
    p = pack_trace([
        {"seq_no": 5, "kind": "ALLOC", "block_id": "x", "size": 10, "stream": 7},
        {"seq_no": 6, "kind": "alloc", "block_id": ("t", 1), "size": 3},
        {"seq_no": 7, "kind": "free", "block_id": "x"},
        {"seq_no": 8, "kind": "resize", "block_id": "x"},
        {"seq_no": 9, "kind": "alloc", "block_id": "y"},
    ])
    assert p.seq_nos == [5, 6, 7, 8, 9]
    assert list(p.reqs["handle"][:3]) == [0, 1, 0]
    ks = p.reqs["kind_stream"]
    assert ks[0] & 3 == _native.KIND_ALLOC and ks[0] >> 2 == 0
    assert ks[1] >> 2 == 1           # stream 0 interned after stream 7
    assert ks[2] & 3 == _native.KIND_FREE
    assert ks[3] & 3 == _native.KIND_UNKNOWN and p.kinds_raw[3] == "resize"
    assert ks[4] & 3 == _native.KIND_MISSING
    assert isinstance(p.host_errors[4], KeyError)


def test_engine_refuses_without_gpu(monkeypatch):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2504_03887_b200 import replay
    from paper_2504_03887_b200.errors import EngineUnavailable
    with pytest.raises(EngineUnavailable):
        replay([{"seq_no": 0, "kind": "alloc", "block_id": 1, "size": 512}])


def test_ingest_library_exports_every_declared_symbol():
    from paper_2504_03887_b200 import _ingest
    header = REPO / "include" / "peakmem_ingest.h"
    assert header_functions(header) == sorted(_ingest.EXPORTED_SYMBOLS)
    if not _ingest.LIB_PATH.exists():
        import __graft_entry__
        __graft_entry__.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_ingest.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pm_\w+)", out))
    for sym in header_functions(header):
        assert sym in exported, sym
    _ingest.load()


def test_wire_pack_roundtrip_and_rejections():
    # pm_wire_pack (host-only): alloc of the next handle -> size word, free
    # -> tag | handle; anything else has no encoding (-> None)
    from paper_2504_03887_b200.allocator import pack_trace
    seq = [{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 700},
           {"seq_no": 1, "kind": "alloc", "block_id": "b", "size": 1 << 40},
           {"seq_no": 2, "kind": "free", "block_id": "a"},
           {"seq_no": 3, "kind": "alloc", "block_id": "c", "size": 1}]
    p = pack_trace(seq)
    offs = np.array([0, len(p.reqs)], dtype=np.int64)
    w = _native.wire_pack(p.reqs, offs)
    assert w is not None
    tag = w >> np.uint64(62)
    assert list(tag) == [0, 0, 1, 0]
    assert list(w[[0, 1, 3]]) == [700, 1 << 40, 1]
    assert int(w[2] & np.uint64(0x7FFFFFFF)) == int(p.reqs["handle"][0])
    for bad in ([{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 5},
                 {"seq_no": 1, "kind": "alloc", "block_id": "b", "size": 5, "stream": 1}],
                [{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 0}],
                [{"seq_no": 0, "kind": "alloc", "block_id": "a", "size": 5},
                 {"seq_no": 1, "kind": "alloc", "block_id": "a", "size": 5}],
                [{"seq_no": 0, "kind": "resize", "block_id": "a", "size": 5}]):
        q = pack_trace(bad)
        assert _native.wire_pack(q.reqs, np.array([0, len(q.reqs)])) is None


def test_wire_pack_threaded_matches_scalar_rule():
    """pm_wire_pack splits traces over host threads: on a multi-million
    request batch every word follows the single-trace rule, and the LOWEST
    bad index is reported whichever thread finds it."""
    from paper_2504_03887_b200 import synth
    reqs, offs = synth.generate(40, first=123)
    w = _native.wire_pack(reqs, offs)
    alloc = (reqs["kind_stream"] & 3) == 0
    assert (w[alloc] == reqs["size"][alloc].astype(np.uint64)).all()
    want_free = np.uint64(1 << 62) | reqs["handle"][~alloc].astype(np.uint64)
    assert (w[~alloc] == want_free).all()
    bad = reqs.copy()
    late, early = int(offs[35]) + 7, int(offs[20]) + 3
    bad["kind_stream"][late] = 2
    bad["kind_stream"][early] = 2
    lib = _native.load_library()
    import ctypes
    out = np.empty(len(bad), np.uint64)
    first = ctypes.c_int64(-1)
    rc = lib.pm_wire_pack(_native._p(bad), _native._p(offs), len(offs) - 1,
                          _native._p(out), ctypes.byref(first))
    assert rc != 0 and first.value == early
