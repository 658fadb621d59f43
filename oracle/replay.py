"""TEST INFRASTRUCTURE -- ctypes wrapper of the C replay oracle.

oracle/replay_oracle.c restates peakmem.allocator (reference
pkg/src/peakmem/allocator.py:155-393) over the same packed records the
engine consumes (include/peakmem_b200.h), so kernel and oracle see
identical inputs.  Built by oracle/Makefile (and __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
LIB_PATH = ORACLE_DIR / "lib" / "liboracle_replay.so"

REQ_DTYPE = np.dtype([("size", "<i8"), ("handle", "<i4"),
                      ("kind_stream", "<u4")])
CFG_DTYPE = np.dtype([(n, "<i8") for n in (
    "k_small_size", "k_small_buffer", "k_min_large_alloc", "k_large_buffer",
    "k_round_large", "alignment", "max_split_size", "device_capacity")])
RESULT_DTYPE = np.dtype([
    ("peak_reserved", "<i8"), ("peak_allocated", "<i8"),
    ("final_reserved", "<i8"), ("final_allocated", "<i8"),
    ("stop_index", "<i8"), ("n_events_replayed", "<i8"),
    ("status", "<i4"), ("n_segments_final", "<i4"),
    ("n_segments_peak", "<i4"), ("max_free_blocks", "<i4")])

_lib = None


def build() -> Path:
    """Compile the oracle with gcc (no GPU needed)."""
    import subprocess
    (ORACLE_DIR / "lib").mkdir(exist_ok=True)
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return LIB_PATH


def load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(LIB_PATH))
        vp = ctypes.c_void_p
        lib.oracle_replay_batch.restype = ctypes.c_int
        lib.oracle_replay_batch.argtypes = [vp, vp, ctypes.c_int32, vp, vp, vp,
                                            vp, ctypes.c_int32]
        lib.pm_synth_counts_ids.argtypes = [vp, ctypes.c_int32, vp, ctypes.c_int]
        lib.pm_synth_fill_ids.argtypes = [vp, ctypes.c_int32, vp, vp, ctypes.c_int]
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(None if a is None else a.ctypes.data)


def replay_batch(reqs: np.ndarray, offsets: np.ndarray, cfgs: np.ndarray,
                 cfg_of: np.ndarray | None = None, timeline: bool = False,
                 n_threads: int | None = None):
    """Replay packed traces on host threads; returns (results, timeline)."""
    lib = load()
    reqs = np.ascontiguousarray(reqs, dtype=REQ_DTYPE)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cfgs = np.ascontiguousarray(cfgs, dtype=CFG_DTYPE)
    if cfg_of is not None:
        cfg_of = np.ascontiguousarray(cfg_of, dtype=np.int32)
    n = len(offsets) - 1
    res = np.zeros(n, dtype=RESULT_DTYPE)
    tl = np.zeros(2 * max(len(reqs), 1), dtype=np.int64) if timeline else None
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    lib.oracle_replay_batch(_p(reqs), _p(offsets), n, _p(cfgs), _p(cfg_of),
                            _p(res), _p(tl), int(n_threads))
    return res, tl


def c3_traces(ids, n_threads: int | None = None):
    """(reqs, offsets) of C3 traces `ids` from the generator compiled into
    this library (workloads/c3gen.c == oracle/c3gen.py), so the reference
    bench arm needs no engine library."""
    lib = load()
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    counts = np.zeros(len(ids), dtype=np.int64)
    lib.pm_synth_counts_ids(_p(ids), len(ids), _p(counts), int(n_threads))
    offs = np.zeros(len(ids) + 1, dtype=np.int64)
    np.cumsum(counts, out=offs[1:])
    reqs = np.empty(int(offs[-1]), dtype=REQ_DTYPE)
    lib.pm_synth_fill_ids(_p(ids), len(ids), _p(offs), _p(reqs), int(n_threads))
    return reqs, offs
