"""Allocator replay API, mirroring peakmem.allocator on the B200 engine.

Reference: pkg/src/peakmem/allocator.py.  Same names, argument meaning and
error behaviour:

  * AllocatorConfig       allocator.py:49-76   (same fields + validation)
  * round_request         allocator.py:79-83
  * segment_size_for      allocator.py:86-92
  * SimulationResult      allocator.py:135-152 (+ segment counts)
  * replay                allocator.py:360-393 (runs on the GPU)
  * load_sequence_file    allocator.py:396-404

plus the batched entry points the engine exists for: `replay_batch` (many
independent request lists, one warp each) and `pack_trace` (the host-side
interning of arbitrary block ids / streams into the 16 B packed records of
include/peakmem_b200.h).

The scalar helpers (round_request, segment_size_for, config validation) are
host-side arithmetic on single Python ints, like the reference's; every
replay runs in the CUDA kernel -- there is no CPU replay path here.
"""

from __future__ import annotations

import math

import json
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native
from ._native import (CFG_DTYPE, KIND_ALLOC, KIND_FREE, KIND_MISSING,
                      KIND_UNKNOWN, REQ_DTYPE)
from .errors import (DoubleFree, DuplicateHandle, EngineLimitExceeded,
                     MalformedSequence, UnknownHandle, ZeroSize)

KIB = 1024
MIB = 1024 * KIB

_INT64_MAX = (1 << 63) - 1


@dataclass(frozen=True)
class AllocatorConfig:
    """Tunable constants of the simulated allocator (allocator.py:49-76).

    max_split_size=None means unbounded (every block may be split);
    device_capacity=None means the device never runs out.
    """

    k_small_size: int = 1 * MIB
    k_small_buffer: int = 2 * MIB
    k_min_large_alloc: int = 10 * MIB
    k_large_buffer: int = 20 * MIB
    k_round_large: int = 2 * MIB
    alignment: int = 512
    max_split_size: int | None = None
    device_capacity: int | None = None

    def __post_init__(self):
        for name in ("k_small_size", "k_small_buffer", "k_min_large_alloc",
                     "k_large_buffer", "k_round_large", "alignment"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.alignment & (self.alignment - 1):
            raise ValueError("alignment must be a power of two")
        if (self.max_split_size is not None
                and self.max_split_size < self.k_large_buffer):
            raise ValueError("max_split_size below the large buffer size")


def round_request(size: int, alignment: int = 512) -> int:
    """Round a request up to the next multiple of the alignment
    (allocator.py:79-83)."""
    if size <= 0:
        raise ZeroSize(f"allocation of {size} bytes")
    return -(-size // alignment) * alignment


def segment_size_for(size: int, cfg: AllocatorConfig = AllocatorConfig()) -> int:
    """Size of the device segment backing a cache miss (allocator.py:86-92)."""
    if size <= cfg.k_small_size:
        return cfg.k_small_buffer
    if size <= cfg.k_min_large_alloc:
        return cfg.k_large_buffer
    return -(-size // cfg.k_round_large) * cfg.k_round_large


@dataclass
class SimulationResult:
    """allocator.py:135-152, plus the engine's segment counts."""

    peak_reserved: int
    peak_allocated: int
    timeline: list[tuple[int, int, int]]
    oom_seq_no: int | None = None
    final_reserved: int = 0
    final_allocated: int = 0
    n_segments_final: int = field(default=0, compare=False)
    n_segments_peak: int = field(default=0, compare=False)

    def to_json_dict(self) -> dict:
        return {
            "peak_reserved": self.peak_reserved,
            "peak_allocated": self.peak_allocated,
            "oom_seq_no": self.oom_seq_no,
            "final_reserved": self.final_reserved,
            "final_allocated": self.final_allocated,
            "timeline": [list(t) for t in self.timeline],
        }


def cfg_record(cfg) -> np.ndarray:
    """One pm_cfg_t from any AllocatorConfig-like object (duck-typed, so the
    reference's own AllocatorConfig works in plugin mode)."""
    rec = np.zeros(1, dtype=CFG_DTYPE)
    for name in ("k_small_size", "k_small_buffer", "k_min_large_alloc",
                 "k_large_buffer", "k_round_large", "alignment"):
        rec[name] = int(getattr(cfg, name))
    ms = getattr(cfg, "max_split_size", None)
    cap = getattr(cfg, "device_capacity", None)
    rec["max_split_size"] = -1 if ms is None else min(int(ms), _INT64_MAX)
    rec["device_capacity"] = -1 if cap is None else min(int(cap), _INT64_MAX)
    return rec


@dataclass
class PackedTrace:
    """One request list interned into packed records.

    seq_nos[i] is the record's own seq_no (need not equal i); host_errors
    maps an index to the exception the reference raises when it reaches
    that record (KeyError for a missing field, ...).
    """

    reqs: np.ndarray
    seq_nos: list
    host_errors: dict[int, BaseException]
    kinds_raw: dict[int, object]


def _int_size(size):
    """The integer the engine replays for a request size, or None.

    round_request (allocator.py:79-83) only compares and ceil-divides the
    size, so a finite float replays like ceil(size): ceil(x / a) ==
    ceil(ceil(x) / a) for an integer alignment a, and size <= 0 iff
    ceil(size) <= 0.  (The reference's timeline then holds floats of the same
    values.)"""
    if isinstance(size, (int, np.integer)) and not isinstance(size, bool):
        return int(size)
    if isinstance(size, (float, np.floating)) and math.isfinite(size):
        return int(math.ceil(size))
    if isinstance(size, bool):
        return int(size)
    return None


def pack_trace(requests: Iterable[dict]) -> PackedTrace:
    """Intern block ids and streams into dense per-trace integers.

    Mirrors the per-request reads of replay() (allocator.py:370-379): the
    kind, then seq_no, then block_id / size / stream.  A read that raises in
    the reference is recorded at its index instead of raised, because the
    reference only raises it if replay reaches that request.
    """
    reqs = list(requests)
    n = len(reqs)
    # Python lists per column, written into the packed records at the end
    # (element-wise numpy writes cost more than the reference's replay)
    sizes = [0] * n
    handles = [0] * n
    ks = [0] * n
    seq_nos: list = [None] * n
    host_errors: dict[int, BaseException] = {}
    kinds_raw: dict[int, object] = {}
    handle_ids: dict = {}
    stream_ids: dict = {}
    for i, req in enumerate(reqs):
        try:
            raw_kind = req["kind"]
            kind = str(raw_kind).lower()
            seq_nos[i] = req["seq_no"]
            if kind == "alloc":
                bid = req["block_id"]
                size = req["size"]
                stream = req.get("stream", 0)
                seen = bid in handle_ids
                h = handle_ids.setdefault(bid, len(handle_ids))
                sid = stream_ids.setdefault(stream, len(stream_ids))
                size = _int_size(size)
                if size is None:
                    if seen:
                        # allocate() checks the handle first (allocator.py:
                        # 274-276): a reused handle is DuplicateHandle whatever
                        # its size -- any positive size lets the kernel say so
                        size = 1
                    else:
                        raise TypeError(
                            f"'<=' not supported for size {req['size']!r}")
                if size > _INT64_MAX:
                    size = 1 << 62  # replays as PM_SIZE_LIMIT
                elif size < -_INT64_MAX:
                    size = -1
                sizes[i] = size
                handles[i] = h
                if sid > 0xFFFF:
                    raise EngineLimitExceeded("more than 65536 streams")
                ks[i] = KIND_ALLOC | (sid << 2)
            elif kind == "free":
                bid = req["block_id"]
                handles[i] = handle_ids.setdefault(bid, len(handle_ids))
                ks[i] = KIND_FREE
            else:
                kinds_raw[i] = raw_kind
                ks[i] = KIND_UNKNOWN
        except Exception as exc:  # surfaced when (if) replay reaches i
            host_errors[i] = exc
            ks[i] = KIND_MISSING
    out = np.zeros(n, dtype=REQ_DTYPE)
    if n:
        out["size"] = sizes
        out["handle"] = handles
        out["kind_stream"] = ks
    return PackedTrace(out, seq_nos, host_errors, kinds_raw)


def _raise_status(status: int, index: int, packed: PackedTrace,
                  code: int = 0) -> None:
    """Re-raise what the reference raises at request `index`
    (allocator.py:371-385): handle errors wrapped in MalformedSequence,
    ZeroSize unwrapped, unknown kinds as MalformedSequence."""
    if status == _native.PM_MISSING_FIELD:
        raise packed.host_errors[index]
    if status == _native.PM_UNKNOWN_KIND:
        raise MalformedSequence(
            f"unknown request kind {packed.kinds_raw[index]!r}")
    if status == _native.PM_ZERO_SIZE:
        raise ZeroSize(f"allocation of {int(packed.reqs['size'][index])} bytes")
    if status == _native.PM_DUPLICATE_HANDLE:
        raise MalformedSequence(str(DuplicateHandle(
            f"handle at request {index} already used")))
    if status == _native.PM_DOUBLE_FREE:
        raise MalformedSequence(str(DoubleFree(
            f"handle at request {index} freed twice")))
    if status == _native.PM_UNKNOWN_HANDLE:
        raise MalformedSequence(str(UnknownHandle(
            f"handle at request {index} never allocated")))
    if status == _native.PM_INVARIANT_VIOLATION:
        raise AssertionError(
            f"allocator invariant violated after request {index}: "
            f"{_native.INVARIANTS.get(code, code)}")
    if status in (_native.PM_SIZE_LIMIT, _native.PM_BAD_STREAM):
        raise EngineLimitExceeded(
            f"request {index} exceeds the engine's packed ranges")
    raise RuntimeError(f"engine status {status} at request {index}")


def _result_from(rec, packed: PackedTrace, timeline: np.ndarray | None,
                 e0: int, result_cls=SimulationResult):
    status = int(rec["status"])
    stop = int(rec["stop_index"])
    oom_seq = None
    if status == _native.PM_OOM:
        oom_seq = packed.seq_nos[stop]
    elif status != _native.PM_OK:
        _raise_status(status, stop, packed, int(rec["max_free_blocks"]))
    n_ok = stop if status == _native.PM_OOM else len(packed.seq_nos)
    tl = []
    if timeline is not None and n_ok:
        pairs = timeline[2 * e0: 2 * (e0 + n_ok)].reshape(-1, 2).tolist()
        tl = [(s, r, a) for s, (r, a) in zip(packed.seq_nos, pairs)]
    kwargs = dict(peak_reserved=int(rec["peak_reserved"]),
                  peak_allocated=int(rec["peak_allocated"]),
                  timeline=tl, oom_seq_no=oom_seq,
                  final_reserved=int(rec["final_reserved"]),
                  final_allocated=int(rec["final_allocated"]))
    res = result_cls(**kwargs)
    try:
        res.n_segments_final = int(rec["n_segments_final"])
        res.n_segments_peak = int(rec["n_segments_peak"])
    except AttributeError:  # a frozen / slotted foreign result class
        pass
    return res


def replay_batch(traces: Sequence[Iterable[dict]],
                 cfgs: AllocatorConfig | Sequence[AllocatorConfig] | None = None,
                 timeline: bool = True,
                 result_cls=SimulationResult, validate: bool = False) -> list:
    """Replay many independent request lists in one kernel launch.

    `cfgs` is one config for all traces or one per trace.  Returns one
    SimulationResult per trace, or raises the first trace's error in the
    reference's convention.  `validate` runs the validating build of the
    kernels, which checks the allocator invariants after every request
    (check_invariants, allocator.py:324-354) and raises AssertionError on a
    violation, as AllocatorState(validate=True) does.
    """
    packed = [pack_trace(t) for t in traces]
    n = len(packed)
    if cfgs is None or not isinstance(cfgs, (list, tuple)):
        cfg_list = [cfgs or AllocatorConfig()]
        cfg_of = None
    else:
        if len(cfgs) != n:
            raise ValueError("need one config per trace")
        cfg_list = list(cfgs)
        cfg_of = np.arange(n, dtype=np.int32)
    cfg_arr = np.concatenate([cfg_record(c) for c in cfg_list])
    lens = np.array([len(p.reqs) for p in packed], dtype=np.int64)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    reqs = (np.concatenate([p.reqs for p in packed]) if n
            else np.zeros(0, dtype=REQ_DTYPE))
    if n == 0:
        return []
    results, tl = _native.replay_host_auto(reqs, offsets, cfg_arr, cfg_of, timeline,
                                           validate=validate)
    return [_result_from(results[i], packed[i], tl, int(offsets[i]), result_cls)
            for i in range(n)]


def replay(requests: Iterable[dict], cfg: AllocatorConfig | None = None,
           validate: bool = False) -> SimulationResult:
    """Apply [{seq_no, kind, block_id, size, stream}] in order
    (allocator.py:360-393) on the GPU.

    OutOfMemory is a verdict, not an error: the result records the failing
    seq_no and the state reached.  Structural problems (free before alloc,
    double free, unknown kind) raise MalformedSequence.  `validate=True`
    checks the allocator invariants after every request on the device
    (allocator.py:291-292, 319-320, 324-354) and raises AssertionError on a
    violation.
    """
    return replay_batch([requests], cfg, validate=validate)[0]


def load_sequence_file(path: str) -> list[dict]:
    """Read the replayable JSON sequence format (allocator.py:396-404)."""
    with open(path, encoding="utf-8") as f:
        data = json.load(f)
    if isinstance(data, dict) and "requests" in data:
        data = data["requests"]
    if not isinstance(data, list):
        raise MalformedSequence("sequence file must hold a list of requests")
    return data
