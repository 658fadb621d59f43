"""Profiling driver: replay N synthetic C3 traces a few times (for ncu).

    python tools/prof_replay.py --traces 600 --launches 2
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=600)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--lib", default=None, help="an alternative build of the engine")
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03887_b200 import synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    if args.lib:
        from paper_2504_03887_b200 import _native
        _native._lib = _native.load_library(args.lib)
    reqs, offs = synth.generate(args.traces, first=args.first)
    batch = DeviceBatch(reqs, offs, cfg_record(AllocatorConfig()))
    for _ in range(args.launches):
        t0 = time.perf_counter()
        batch.launch()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        res = batch.results()
        ev = int(res["n_events_replayed"].sum())
        ctl = batch.d_ws[:64].cpu().numpy().view(np.uint32)
        print(f"retries: narrow passes {ctl[9:12].tolist()}, wide tiers {ctl[12:16].tolist()}")
        print(f"{args.traces} traces {ev} events {dt*1e3:.1f} ms "
              f"{ev/dt/1e9:.3f} Gev/s maxF {res['max_free_blocks'].max()} "
              f"status {set(res['status'].tolist())}")


if __name__ == "__main__":
    main()
