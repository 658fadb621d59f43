"""BASELINE configs[1] / SURVEY §8d C2: GPT-2 small training traces at batch
sizes 1..64, replayed as 64 independent traces on one B200.

    python tools/bench_c2.py [--traces DIR] [--ref-sample 8]

1. replay: the 64 orchestrated sequences (tests/golden/c2_sweep.npz) as ONE
   batch -- device-resident (DeviceBatch / pm_replay_batch, CUDA events,
   median of 20 launches) and through the host C ABI (pm_replay_host with
   timeline, wall clock) -- every result and timeline bit-exact against the
   reference (tests/golden/c2_sweep_golden.json).
2. end to end (when DIR holds gpt2_bs{b}_s128.trace.json.gz + .sidecar.json):
   file -> parse_trace -> PeakMemoryEstimator.estimate for all 64 traces,
   reports compared byte for byte with the reference's; the reference
   package itself (baseline/_ref) timed on --ref-sample of the files on the
   same host.
Prints one JSON line.
"""

from __future__ import annotations

import argparse
import gzip
import json
import statistics
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", default=str(REPO / "c2cache"))
    ap.add_argument("--ref-sample", type=int, default=8)
    args = ap.parse_args()
    import logging
    logging.disable(logging.WARNING)
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    from paper_2504_03887_b200 import _native
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    from test_captures import c2_sweep, check_sweep

    reqs, offs, meta = c2_sweep()
    cfg = cfg_record(AllocatorConfig())
    out = {"config": "C2: GPT-2 small (124M) training traces, batch 1..64 x seq 128, "
                     "AdamW, iterations=2: 64 independent traces on 1 B200",
           "traces": 64, "requests": int(offs[-1])}
    # --- replay, device resident --------------------------------------------
    b = DeviceBatch(reqs, offs, cfg)
    for _ in range(3):
        b.launch()
    torch.cuda.synchronize()
    ms = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.launch()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    check_sweep(b.results(), None, offs, meta)
    t = statistics.median(ms) / 1e3
    out["replay_device"] = {"ms": t * 1e3, "events_per_s": int(offs[-1]) / t}
    # --- replay through the host C ABI, with the full timeline ---------------
    _native.replay_host(reqs, offs, cfg, None, True)
    t0 = time.perf_counter()
    res, tl = _native.replay_host(reqs, offs, cfg, None, True)
    th = time.perf_counter() - t0
    check_sweep(res, tl, offs, meta)
    out["replay_host_abi"] = {"ms": th * 1e3, "events_per_s": int(offs[-1]) / th,
                              "api": "pm_replay_host, pageable host buffers, timeline on"}
    out["parity"] = "64/64 traces bit-exact vs the reference (peaks, finals, segment counts, timelines)"

    # --- end to end: 64 files -> 64 reports ----------------------------------
    src = Path(args.traces)
    if (src / "gpt2_bs1_s128.trace.json.gz").exists():
        tmp = Path(tempfile.mkdtemp())
        files = []
        for m in meta:
            tr = tmp / f"{m['name']}.json"
            tr.write_bytes(gzip.open(src / f"{m['name']}.trace.json.gz").read())
            files.append((tr, src / f"{m['name']}.sidecar.json", m))
        # warm-up (CUDA context, pools, libraries)
        eng.PeakMemoryEstimator().estimate(
            eng.parse_trace(files[0][0], sidecar=eng.load_sidecar(files[0][1])))
        t0 = time.perf_counter()
        reports = [eng.PeakMemoryEstimator().estimate(
            eng.parse_trace(tr, sidecar=eng.load_sidecar(sc))) for tr, sc, _ in files]
        te = time.perf_counter() - t0
        same = sum(r.canonical_json() == m["report"] for r, (_, _, m) in zip(reports, files))
        mb = sum(tr.stat().st_size for tr, _, _ in files) / 1e6
        out["e2e_engine"] = {"s": te, "traces_per_s": 64 / te, "json_mb": round(mb, 1),
                             "reports_identical": f"{same}/64"}
        ref_root = REPO / "baseline" / "_ref"
        if (ref_root / "peakmem").exists() and args.ref_sample:
            sys.path.insert(0, str(ref_root))
            import peakmem as ref
            pick = files[:: max(1, 64 // args.ref_sample)][: args.ref_sample]
            t0 = time.perf_counter()
            for tr, sc, m in pick:
                r = ref.PeakMemoryEstimator().estimate(
                    ref.parse_trace(str(tr), sidecar=ref.load_sidecar(str(sc))))
                assert r.canonical_json() == m["report"]
            tr_s = (time.perf_counter() - t0) / len(pick)
            out["e2e_reference"] = {"s_per_trace": tr_s, "sample": len(pick),
                                    "extrapolated_64_s": 64 * tr_s, "cores": 1,
                                    "speedup_engine_vs_reference": 64 * tr_s / te}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
