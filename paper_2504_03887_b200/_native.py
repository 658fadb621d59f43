"""ctypes binding of the engine's C ABI (include/peakmem_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` into
paper_2504_03887_b200/lib/.  There is no CPU fallback: if the library or a
CUDA device is missing, every entry point raises EngineUnavailable.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import EngineUnavailable

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = LIB_DIR / "libpeakmem_b200.so"
# the same kernels built with -DPM_VALIDATE: replay(validate=True)
VALIDATE_LIB_PATH = LIB_DIR / "libpeakmem_b200_validate.so"

# --- packed layouts (must match include/peakmem_b200.h) --------------------

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
assert REQ_DTYPE.itemsize == 16 and CFG_DTYPE.itemsize == 64
assert RESULT_DTYPE.itemsize == 64

KIND_ALLOC, KIND_FREE, KIND_UNKNOWN, KIND_MISSING = 0, 1, 2, 3

(PM_OK, PM_OOM, PM_UNKNOWN_HANDLE, PM_DOUBLE_FREE, PM_DUPLICATE_HANDLE,
 PM_ZERO_SIZE, PM_UNKNOWN_KIND, PM_MISSING_FIELD, PM_BAD_HANDLE,
 PM_SIZE_LIMIT, PM_BAD_STREAM, PM_POOL_OVERFLOW, PM_ENCODING_LIMIT,
 PM_INVARIANT_VIOLATION) = range(14)

#: pm_invariant_t (include/peakmem_b200.h) -> the check_invariants assertion
#: it restates (allocator.py:324-354)
INVARIANTS = {1: "blk.size > 0", 2: "unaligned block",
              3: "tiling gap/overlap or broken back-link",
              4: "adjacent free blocks", 5: "blocks do not tile segment",
              6: "conservation", 7: "allocated_total == allocated_bytes",
              8: "pool and segment chains disagree",
              9: "reserved_bytes <= device_capacity",
              10: "neighbouring blocks on different streams"}

#: every symbol include/peakmem_b200.h declares
EXPORTED_SYMBOLS = ("pm_last_error", "pm_version", "pm_validate_inject",
                    "pm_replay_workspace_bytes",
                    "pm_replay_batch", "pm_replay_host", "pm_wire_pack",
                    "pm_replay_host_wire",
                    "pm_capacity_workspace_bytes", "pm_capacity_search")

_lib = None
_vlib = None


def _p(arr) -> ctypes.c_void_p:
    """Host pointer of a contiguous numpy array (None -> NULL)."""
    if arr is None:
        return ctypes.c_void_p(None)
    return ctypes.c_void_p(arr.ctypes.data)


def load_library(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and prototype the engine library; raise if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise EngineUnavailable(
            f"engine library {p} is not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(str(p))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.pm_last_error.restype = ctypes.c_char_p
    lib.pm_last_error.argtypes = []
    lib.pm_version.restype = ctypes.c_int
    lib.pm_version.argtypes = []
    lib.pm_validate_inject.restype = ctypes.c_int
    lib.pm_validate_inject.argtypes = [i64, i32]
    lib.pm_replay_workspace_bytes.restype = ctypes.c_int
    lib.pm_replay_workspace_bytes.argtypes = [
        i64, i64, i32, ctypes.POINTER(ctypes.c_size_t)]
    lib.pm_replay_batch.restype = ctypes.c_int
    lib.pm_replay_batch.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp, vp,
                                    ctypes.c_size_t, i64, i64, vp]
    lib.pm_replay_host.restype = ctypes.c_int
    lib.pm_replay_host.argtypes = [vp, vp, i32, vp, i32, vp, vp, vp, vp]
    lib.pm_replay_host_wire.restype = ctypes.c_int
    lib.pm_replay_host_wire.argtypes = [vp, vp, i32, vp, i32, vp, vp, vp, vp]
    lib.pm_wire_pack.restype = ctypes.c_int
    lib.pm_wire_pack.argtypes = [vp, vp, i32, vp, ctypes.POINTER(i64)]
    lib.pm_capacity_workspace_bytes.restype = ctypes.c_int
    lib.pm_capacity_workspace_bytes.argtypes = [
        i64, i64, i32, ctypes.POINTER(ctypes.c_size_t)]
    lib.pm_capacity_search.restype = ctypes.c_int
    lib.pm_capacity_search.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp, vp, vp,
                                       vp, i32, vp, ctypes.c_size_t, i64, i64,
                                       vp]
    if path is None:
        _lib = lib
    return lib


def load_validate_library() -> ctypes.CDLL:
    """The validating build of the engine (same ABI, -DPM_VALIDATE)."""
    global _vlib
    if _vlib is None:
        if not VALIDATE_LIB_PATH.exists():
            raise EngineUnavailable(
                f"validating engine library {VALIDATE_LIB_PATH} is not built; "
                "run __graft_entry__.build()")
        _vlib = load_library(VALIDATE_LIB_PATH)
    return _vlib


def check(rc: int, lib=None) -> None:
    if rc != 0:
        lib = lib or load_library()
        msg = lib.pm_last_error().decode(errors="replace")
        raise RuntimeError(f"peakmem_b200 engine error {rc}: {msg}")


def require_device() -> None:
    """Fail loudly unless a CUDA device is present (no CPU fallback)."""
    if os.environ.get("PEAKMEM_B200_SKIP_DEVICE_CHECK"):
        return
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is part of the image
        return
    if not torch.cuda.is_available():
        raise EngineUnavailable(
            "no CUDA device: the B200 engine has no CPU fallback")


def workspace_bytes(total_events: int, max_trace_events: int,
                    n_traces: int) -> int:
    lib = load_library()
    out = ctypes.c_size_t(0)
    check(lib.pm_replay_workspace_bytes(total_events, max_trace_events,
                                        n_traces, ctypes.byref(out)), lib)
    return int(out.value)


def replay_host(reqs: np.ndarray, offsets: np.ndarray, cfgs: np.ndarray,
                cfg_of: np.ndarray | None, want_timeline: bool,
                stream: int = 0, validate: bool = False):
    """Host-buffer replay through pm_replay_host (H2D + kernel + D2H)."""
    lib = load_validate_library() if validate else load_library()
    require_device()
    reqs = np.ascontiguousarray(reqs, dtype=REQ_DTYPE)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cfgs = np.ascontiguousarray(cfgs, dtype=CFG_DTYPE)
    n_traces = len(offsets) - 1
    if cfg_of is not None:
        cfg_of = np.ascontiguousarray(cfg_of, dtype=np.int32)
    results = np.zeros(n_traces, dtype=RESULT_DTYPE)
    timeline = (np.zeros(2 * max(len(reqs), 1), dtype=np.int64)
                if want_timeline else None)
    check(lib.pm_replay_host(_p(reqs), _p(offsets), n_traces, _p(cfgs),
                             len(cfgs), _p(cfg_of), _p(results),
                             _p(timeline), ctypes.c_void_p(stream)), lib)
    return results, timeline


def wire_pack(reqs: np.ndarray, offsets: np.ndarray, out: np.ndarray | None = None):
    """Pack pm_req_t traces into 8-byte wire words (include/peakmem_b200.h).

    Returns the uint64 words, or None when some request has no wire
    encoding (the caller then replays the pm_req_t records).  Host-only."""
    lib = load_library()
    reqs = np.ascontiguousarray(reqs, dtype=REQ_DTYPE)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    if out is None:
        out = np.empty(len(reqs), dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    rc = lib.pm_wire_pack(_p(reqs), _p(offsets), len(offsets) - 1, _p(out),
                          ctypes.byref(bad))
    if rc != 0:
        if bad.value >= 0:
            return None
        check(rc, lib)
    return out[:len(reqs)]


def replay_host_wire(words: np.ndarray, offsets: np.ndarray, cfgs: np.ndarray,
                     cfg_of: np.ndarray | None, want_timeline: bool,
                     stream: int = 0, validate: bool = False):
    """Host-buffer replay of wire words through pm_replay_host_wire."""
    lib = load_validate_library() if validate else load_library()
    require_device()
    words = np.ascontiguousarray(words, dtype=np.uint64)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cfgs = np.ascontiguousarray(cfgs, dtype=CFG_DTYPE)
    n_traces = len(offsets) - 1
    if cfg_of is not None:
        cfg_of = np.ascontiguousarray(cfg_of, dtype=np.int32)
    results = np.zeros(n_traces, dtype=RESULT_DTYPE)
    timeline = (np.zeros(2 * max(len(words), 1), dtype=np.int64)
                if want_timeline else None)
    check(lib.pm_replay_host_wire(_p(words), _p(offsets), n_traces, _p(cfgs),
                                  len(cfgs), _p(cfg_of), _p(results),
                                  _p(timeline), ctypes.c_void_p(stream)), lib)
    return results, timeline


def replay_host_auto(reqs: np.ndarray, offsets: np.ndarray, cfgs: np.ndarray,
                     cfg_of: np.ndarray | None, want_timeline: bool,
                     stream: int = 0, validate: bool = False):
    """pm_replay_host_wire when every request has a wire encoding (half the
    H2D bytes), else pm_replay_host; results are identical."""
    words = wire_pack(reqs, offsets) if len(reqs) else None
    if words is not None:
        return replay_host_wire(words, offsets, cfgs, cfg_of, want_timeline,
                                stream, validate)
    return replay_host(reqs, offsets, cfgs, cfg_of, want_timeline, stream,
                       validate)
