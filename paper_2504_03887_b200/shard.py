"""Sharding independent traces over GPUs.

Traces never interact, so N GPUs each replay a disjoint shard -- no
collective on the data path.  Greedy LPT on trace length (longest trace to
the least-loaded rank) keeps the per-rank work within one trace of even;
the only cross-rank traffic is the timing reduction (max over ranks) and,
optionally, a gather of the 64 B per-trace results.
"""

from __future__ import annotations

import numpy as np


def lpt_shards(lengths: np.ndarray, world: int) -> list[np.ndarray]:
    """Trace ids per rank (each sorted ascending), greedy LPT."""
    lengths = np.asarray(lengths, dtype=np.int64)
    order = np.argsort(-lengths, kind="stable")
    loads = np.zeros(world, dtype=np.int64)
    parts: list[list[int]] = [[] for _ in range(world)]
    for t in order.tolist():
        r = int(np.argmin(loads))
        parts[r].append(t)
        loads[r] += lengths[t]
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def gather_results(local_results: np.ndarray, local_ids: np.ndarray,
                   n_traces: int, dist=None) -> np.ndarray:
    """Reassemble per-trace result records on every rank (host gather of
    the 64 B results; the only cross-device step of a sweep)."""
    if dist is None:
        out = np.zeros(n_traces, dtype=local_results.dtype)
        out[local_ids] = local_results
        return out
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (local_ids.tolist(), local_results.tobytes()))
    out = np.zeros(n_traces, dtype=local_results.dtype)
    for ids, blob in parts:
        out[np.asarray(ids, dtype=np.int64)] = np.frombuffer(
            blob, dtype=local_results.dtype)
    return out
