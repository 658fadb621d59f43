"""A sweep made only of fragmented traces: C5-style
event-level traces (synth_events) orchestrated into request sequences whose
free blocks outgrow the main pass's register directory, replayed as one
batch.  Every trace leaves the main pass mid-way, continues from its
checkpoint in the multi-warp shared-memory pass 1 (or later passes), and
must equal the oracle.

    python tools/bench_frag.py [--leaves 600] [--traces 3552]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10000)
    ap.add_argument("--traces", type=int, default=3552)
    ap.add_argument("--variants", type=int, default=16)
    ap.add_argument("--check", type=int, default=64, help="traces checked vs the oracle")
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    from oracle import replay as oracle
    seqs = []
    for v in range(args.variants):
        b = synth_events.generate(args.leaves + 37 * v, 2, seed=7 + v)
        seqs.append(api.build_sequence(api.analyze(b), 2).packed)
    parts = [seqs[i % len(seqs)] for i in range(args.traces)]
    offs = np.zeros(len(parts) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=offs[1:])
    reqs = np.concatenate(parts)
    cfg = cfg_record(AllocatorConfig())
    b = DeviceBatch(reqs, offs, cfg)
    b.launch()
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.launch()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    res = b.results()
    ev = int(res["n_events_replayed"].sum())
    k = min(args.check, len(parts))
    want, _ = oracle.replay_batch(reqs[:offs[k]], offs[:k + 1], cfg)
    print(json.dumps({
        "workload": f"{args.traces} fragmented C5-style traces ({args.variants} variants, "
                    f"~{args.leaves} leaves, 2 iterations)",
        "requests": ev, "ms": min(ms), "events_per_s": ev / (min(ms) / 1e3),
        "max_free_blocks": int(res["max_free_blocks"].max()),
        "median_free_blocks": int(np.median(res["max_free_blocks"])),
        "retry_passes": b.tier_counts(),
        "oracle_equal_first": int(k) if (res[:k] == want).all() else "MISMATCH"}))


if __name__ == "__main__":
    main()
