"""TEST INFRASTRUCTURE -- CPU restatement of the batched capacity bisection
(pm_capacity_search, include/peakmem_b200.h).

Each probe is the C replay oracle (oracle/replay_oracle.c, restating
allocator.py:155-393) at AllocatorConfig(device_capacity=C).  The bracket
and unit follow from allocator.py:86-92 (segment sizes) and :258-287,
:328-333 (the only reads of device_capacity): see the header.
`linear_scan` is the brute-force definition used to pin the bisection on
small traces.
"""

from __future__ import annotations

from math import gcd

import numpy as np

from . import replay as oracle

UNBOUNDED = -1


def _unit(cfg) -> int:
    return gcd(gcd(int(cfg["k_small_buffer"]), int(cfg["k_large_buffer"])),
               int(cfg["k_round_large"]))


def _cfg_of_trace(cfgs, cfg_of, n):
    return [cfgs[cfg_of[t] if cfg_of is not None else 0].copy() for t in range(n)]


def _replay_subset(reqs, offsets, tcfgs, traces):
    sub = [reqs[offsets[t]:offsets[t + 1]] for t in traces]
    offs = np.zeros(len(traces) + 1, np.int64)
    np.cumsum([len(x) for x in sub], out=offs[1:])
    cfg_arr = np.array([tcfgs[t] for t in traces], dtype=oracle.CFG_DTYPE)
    res, _ = oracle.replay_batch(np.concatenate(sub) if sub else reqs[:0], offs,
                                 cfg_arr, np.arange(len(traces), dtype=np.int32))
    return res


def bisect(reqs, offsets, cfgs, cfg_of=None, max_rounds: int = 64):
    """-> dict like DeviceBatch.capacity_search (lists of probes per trace)."""
    n = len(offsets) - 1
    tcfgs = _cfg_of_trace(cfgs, cfg_of, n)
    for c in tcfgs:
        c["device_capacity"] = UNBOUNDED
    r0 = _replay_subset(reqs, offsets, tcfgs, list(range(n)))
    lo = [0] * n
    hi = [0] * n
    unit = [_unit(c) for c in tcfgs]
    min_cap = [0] * n
    for t in range(n):
        if int(r0[t]["status"]) != 0:
            min_cap[t] = -1
            continue
        pa, pr = int(r0[t]["peak_allocated"]), int(r0[t]["peak_reserved"])
        # allocated is capacity-independent only when every block splits
        split_all = int(tcfgs[t]["max_split_size"]) < 0
        lo[t] = (pa - 1) // unit[t] if (pa > 0 and split_all) else -1
        hi[t] = pr // unit[t]
    probes = [[] for _ in range(n)]
    for _ in range(max_rounds):
        active = [t for t in range(n) if min_cap[t] == 0 and hi[t] - lo[t] > 1]
        if not active:
            break
        for t in active:
            tcfgs[t]["device_capacity"] = (lo[t] + (hi[t] - lo[t]) // 2) * unit[t]
        res = _replay_subset(reqs, offsets, tcfgs, active)
        for t, r in zip(active, res):
            cap = int(tcfgs[t]["device_capacity"])
            probes[t].append((cap, r.copy()))
            if int(r["status"]) == 1:
                lo[t] = cap // unit[t]
            elif int(r["status"]) == 0:
                hi[t] = cap // unit[t]
            else:
                min_cap[t] = -2
    for t in range(n):
        if min_cap[t] == 0:
            min_cap[t] = hi[t] * unit[t]
    return {"min_capacity": min_cap, "unbounded": r0, "probes": probes}


def linear_scan(reqs, offsets, cfg, t: int):
    """Smallest multiple of the unit in [0, peak_reserved] that runs, and
    whether runnability was monotone over that range."""
    tc = [cfg.copy()]
    tc[0]["device_capacity"] = UNBOUNDED
    sub = reqs[offsets[t]:offsets[t + 1]]
    offs = np.array([0, len(sub)], np.int64)
    r0, _ = oracle.replay_batch(sub, offs, np.array(tc, dtype=oracle.CFG_DTYPE))
    u = _unit(cfg)
    pa, pr = int(r0[0]["peak_allocated"]), int(r0[0]["peak_reserved"])
    del pa
    ks = list(range(0, pr // u + 1))
    cfg_arr = np.array([cfg] * len(ks), dtype=oracle.CFG_DTYPE)
    cfg_arr["device_capacity"] = np.array(ks, np.int64) * u
    reps = np.tile(sub, len(ks))
    offs = np.arange(len(ks) + 1, dtype=np.int64) * len(sub)
    res, _ = oracle.replay_batch(reps, offs, cfg_arr,
                                 np.arange(len(ks), dtype=np.int32))
    ok = [int(r["status"]) == 0 for r in res]
    first = next(i for i, v in enumerate(ok) if v)
    monotone = all(ok[first:])
    return ks[first] * u, monotone
