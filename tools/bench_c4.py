"""Time the C4 config sweep: 8 GPT-2 capture sequences + 42 C3
traces, each under the 69 allocator configs, as one device-resident batch.

    python tools/bench_c4.py [--c3 42] [--check]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", type=int, default=42)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--lib", default=None, help="an alternative build of the engine")
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from c4_cases import c4_batch, c4_configs
    from paper_2504_03887_b200 import synth
    from paper_2504_03887_b200.engine import DeviceBatch
    if args.lib:
        from paper_2504_03887_b200 import _native
        _native._lib = _native.load_library(args.lib)
    z = np.load(ROOT / "tests" / "golden" / "c2_sequences.npz")
    r3, o3 = synth.generate(args.c3, first=9000)
    reqs = np.concatenate([z["reqs"], r3])
    offs = np.concatenate([z["offsets"], o3[1:] + z["offsets"][-1]])
    cfgs = c4_configs()
    big, boffs, rec, cfg_of = c4_batch(reqs, offs, cfgs)
    b = DeviceBatch(big, boffs, rec, cfg_of)
    b.launch()
    torch.cuda.synchronize()
    times, dev_ms = [], []
    for _ in range(args.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        b.launch()
        e1.record()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        dev_ms.append(round(e0.elapsed_time(e1), 2))
    res = b.results()
    ev = int(res["n_events_replayed"].sum())
    line = {"workload": "C4", "traces": len(offs) - 1, "configs": len(cfgs),
            "replays": len(boffs) - 1, "requests": ev, "seconds": min(times),
            "events_per_s": ev / min(times),
            "device_ms": dev_ms, "wall_ms": [round(t * 1e3, 2) for t in times],
            "statuses": sorted(set(res["status"].tolist())),
            "retry_passes": b.tier_counts(),
            "max_free_blocks": int(res["max_free_blocks"].max()),
            "longest_trace": int(np.diff(boffs).max())}
    if args.check:
        from oracle import replay as oracle
        t0 = time.perf_counter()
        want, _ = oracle.replay_batch(big, boffs, rec, cfg_of)
        line["oracle_s"] = time.perf_counter() - t0
        line["oracle_equal"] = bool(all((res[f] == want[f]).all() for f in want.dtype.names))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
