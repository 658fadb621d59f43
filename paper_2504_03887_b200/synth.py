"""Synthetic request-level traces for sweeps and benchmarks.

Thin ctypes wrapper of workloads/c3gen.c (host C, pthreads): Llama-style
training traces of ~1e5 requests each, trace i drawn from numpy's
Generator(PCG64(1_000_003 + i)) exactly as the spec oracle/c3gen.py does,
emitted directly in the engine's packed record format.
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
        i32, ci = ctypes.c_int32, ctypes.c_int
        lib.pm_synth_counts.argtypes = [i32, i32, vp, ci]
        lib.pm_synth_fill.argtypes = [i32, i32, vp, vp, ci]
        lib.pm_synth_counts_ids.argtypes = [vp, i32, vp, ci]
        lib.pm_synth_fill_ids.argtypes = [vp, i32, vp, vp, ci]
        _lib = lib
    return _lib


def _threads(n):
    return len(os.sched_getaffinity(0)) if n is None else n


def counts(ids: np.ndarray, n_threads: int | None = None) -> np.ndarray:
    """Request count of every trace in `ids`."""
    lib = _load()
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    out = np.zeros(len(ids), dtype=np.int64)
    lib.pm_synth_counts_ids(ids.ctypes.data, len(ids), out.ctypes.data,
                            _threads(n_threads))
    return out


def generate_ids(ids: np.ndarray, n_threads: int | None = None,
                 out: np.ndarray | None = None, lengths: np.ndarray | None = None):
    """(reqs, offsets) for the traces `ids`, in that order."""
    lib = _load()
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    if lengths is None:
        lengths = counts(ids, n_threads)
    offsets = np.zeros(len(ids) + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    total = int(offsets[-1])
    if out is None:
        out = np.empty(total, dtype=REQ_DTYPE)
    elif len(out) < total:
        raise ValueError("output buffer too small")
    lib.pm_synth_fill_ids(ids.ctypes.data, len(ids), offsets.ctypes.data,
                          out.ctypes.data, _threads(n_threads))
    return out[:total], offsets


def generate(n_traces: int, first: int = 0, n_threads: int | None = None,
             out: np.ndarray | None = None):
    """Return (reqs, offsets) for traces first .. first+n_traces-1.

    `out` may be a preallocated (e.g. pinned) buffer viewed as REQ_DTYPE."""
    return generate_ids(np.arange(first, first + n_traces), n_threads, out)
