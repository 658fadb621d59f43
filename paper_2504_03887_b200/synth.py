"""Synthetic request-level traces for sweeps and benchmarks.

Thin ctypes wrapper of csrc/synth.c (host C, pthreads): Llama-style training
traces of ~1e5 requests each, seeded 1_000_003 + i, emitted directly in the
engine's packed record format.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from ._native import LIB_DIR, REQ_DTYPE

SYNTH_LIB = LIB_DIR / "libpeakmem_synth.so"
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not SYNTH_LIB.exists():
            raise RuntimeError(f"{SYNTH_LIB} not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(SYNTH_LIB))
        vp = ctypes.c_void_p
        lib.pm_synth_counts.argtypes = [ctypes.c_int32, ctypes.c_int32, vp, ctypes.c_int]
        lib.pm_synth_fill.argtypes = [ctypes.c_int32, ctypes.c_int32, vp, vp, ctypes.c_int]
        _lib = lib
    return _lib


def generate(n_traces: int, first: int = 0, n_threads: int | None = None,
             out: np.ndarray | None = None):
    """Return (reqs, offsets) for traces first .. first+n_traces-1.

    `out` may be a preallocated (e.g. pinned) buffer viewed as REQ_DTYPE."""
    lib = _load()
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    counts = np.zeros(n_traces, dtype=np.int64)
    lib.pm_synth_counts(first, n_traces, counts.ctypes.data, n_threads)
    offsets = np.zeros(n_traces + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    total = int(offsets[-1])
    if out is None:
        out = np.empty(total, dtype=REQ_DTYPE)
    elif len(out) < total:
        raise ValueError("output buffer too small")
    lib.pm_synth_fill(first, n_traces, offsets.ctypes.data, out.ctypes.data,
                      n_threads)
    return out[:total], offsets
