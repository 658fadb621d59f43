"""Time the batched capacity bisection (pm_capacity_search) on C3 traces.

    python tools/bench_capacity.py --traces 10000 [--check 100]

Prints one JSON line: traces, rounds, probe replays, replayed requests,
wall time, requests/s over all probes, mean capacity saving vs the unbounded
peak; --check K compares the first K traces with the CPU oracle bisection.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=10000)
    ap.add_argument("--check", type=int, default=0)
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03887_b200 import synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    reqs, offs = synth.generate(args.traces)
    cfg = cfg_record(AllocatorConfig())
    b = DeviceBatch(reqs, offs, cfg)
    b.launch()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = b.capacity_search()
    t1 = time.perf_counter()
    lens = np.diff(offs)
    probes = out["n_probes"].astype(np.int64)
    replayed = int(lens.sum() + (lens * probes).sum())
    peak = out["unbounded"]["peak_reserved"].astype(np.int64)
    mc = out["min_capacity"]
    line = {"traces": args.traces, "requests": int(lens.sum()),
            "rounds": int(probes.max()), "probe_replays": int(probes.sum()),
            "replayed_requests": replayed, "seconds": t1 - t0,
            "replayed_requests_per_s": replayed / (t1 - t0),
            "mean_saving_frac": float(np.mean((peak - mc) / peak)),
            "traces_saving": int((mc < peak).sum())}
    if args.check:
        from oracle import capacity as ocap
        k = args.check
        sub_offs = offs[:k + 1]
        want = ocap.bisect(reqs[:sub_offs[-1]], sub_offs, cfg)
        line["check_traces"] = k
        line["check_equal"] = bool(list(mc[:k]) == list(want["min_capacity"]) and
                                   all(int(probes[t]) == len(want["probes"][t])
                                       for t in range(k)))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
