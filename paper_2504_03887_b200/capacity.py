"""Batched capacity bisection: the smallest
`AllocatorConfig.device_capacity` each request sequence replays in without
OutOfMemory, for many sequences at once on the GPU.

The reference answers "how much memory does this job need" with the
unbounded run's peak_reserved (estimator.py:155; pkg/README.md:12-13).  With
a finite capacity its allocator releases cached segments under pressure
(allocator.py:258-287), so a job can run in less than that peak; this finds
how much less, replaying every sequence at its own bisection midpoint per
round (`pm_capacity_search`, include/peakmem_b200.h).  Each probe is exactly
the reference's replay() at AllocatorConfig(device_capacity=C).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native
from .allocator import (AllocatorConfig, _raise_status, cfg_record, pack_trace)
from .engine import DeviceBatch


@dataclass
class CapacityResult:
    """min_capacity: smallest runnable capacity found (a multiple of
    gcd(k_small_buffer, k_large_buffer, k_round_large)); unbounded_peak:
    the reference's estimate (peak_reserved with no capacity); probes:
    [(capacity, oom_seq_no or None)] in bisection order."""

    min_capacity: int
    unbounded_peak: int
    peak_allocated: int
    probes: list = field(default_factory=list)

    @property
    def saving(self) -> int:
        return self.unbounded_peak - self.min_capacity


def min_runnable_capacity(sequences: Sequence[Iterable[dict]],
                          cfgs: AllocatorConfig | Sequence[AllocatorConfig] | None = None,
                          max_probes: int = 64) -> list[CapacityResult]:
    """Bisect each sequence's smallest runnable capacity (device_capacity in
    the configs is ignored).  Malformed sequences raise like replay()."""
    packed = [pack_trace(t) for t in sequences]
    n = len(packed)
    if n == 0:
        return []
    if cfgs is None or not isinstance(cfgs, (list, tuple)):
        cfg_arr = cfg_record(cfgs or AllocatorConfig())
        cfg_of = None
    else:
        if len(cfgs) != n:
            raise ValueError("need one config per sequence")
        cfg_arr = np.concatenate([cfg_record(c) for c in cfgs])
        cfg_of = np.arange(n, dtype=np.int32)
    lens = np.array([len(p.reqs) for p in packed], dtype=np.int64)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    out = DeviceBatch(reqs, offsets, cfg_arr, cfg_of).capacity_search(max_probes)
    results = []
    for i, p in enumerate(packed):
        u = out["unbounded"][i]
        if int(u["status"]) != _native.PM_OK:
            _raise_status(int(u["status"]), int(u["stop_index"]), p)
        probes = []
        for k in range(min(int(out["n_probes"][i]), max_probes)):
            r = out["probe_results"][k, i]
            oom = (p.seq_nos[int(r["stop_index"])]
                   if int(r["status"]) == _native.PM_OOM else None)
            probes.append((int(out["probe_capacity"][k, i]), oom))
        results.append(CapacityResult(
            min_capacity=int(out["min_capacity"][i]),
            unbounded_peak=int(u["peak_reserved"]),
            peak_allocated=int(u["peak_allocated"]), probes=probes))
    return results


__all__ = ["CapacityResult", "min_runnable_capacity"]
