"""Goldens for SURVEY §8d C2: GPT-2 small (124M) training traces at batch
sizes 1..64 (sequence length 128, AdamW, 3 profiled iterations), captured
offline by tools/capture_models.py (recipe: reference capture.py:79-85) into
data/captures/gpt2_bs{b}_s128 (not committed: ~25 MB of JSON each).

Run where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_c2.py

For every batch size the REFERENCE runs the whole pipeline
(parse_trace -> PeakMemoryEstimator.estimate, iterations=2) and its replay
with segment instrumentation (make_golden.run_reference on
build_sequence(analyze(bundle), 2).replay_records()).  Writes
tests/golden/c2_sweep.npz (the 64 packed request sequences) and
tests/golden/c2_sweep_golden.json (per trace: replay results incl. segment
counts and timeline digest, the report bytes, the reference's own
end-to-end time on this host).
"""

from __future__ import annotations

import hashlib
import json
import logging
import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))
logging.disable(logging.WARNING)

CAPS = REPO / "data" / "captures"
BATCHES = list(range(1, 65))


def one(b):
    from peakmem import PeakMemoryEstimator, load_sidecar, parse_trace
    from peakmem.allocator import AllocatorConfig
    from peakmem.orchestration import analyze, build_sequence
    from make_golden import run_reference
    from paper_2504_03887_b200.allocator import pack_trace
    src = CAPS / f"gpt2_bs{b}_s128"
    t0 = time.perf_counter()
    side = load_sidecar(str(src / "sidecar.json"))
    bundle = parse_trace(str(src / "trace.json"), sidecar=side)
    report = PeakMemoryEstimator().estimate(bundle)
    e2e = time.perf_counter() - t0
    recs = build_sequence(analyze(bundle), iterations=2).replay_records()
    res = run_reference(recs, AllocatorConfig())
    p = pack_trace(recs)
    return {"batch": b, "name": src.name, "n_events": len(bundle.events),
            "trace_sha256": hashlib.sha256((src / "trace.json").read_bytes()).hexdigest(),
            "report": report.canonical_json(), "reference_e2e_s": e2e,
            "n_requests": len(recs), **res}, p.reqs


def main():
    with mp.get_context("fork").Pool(4) as pool:
        out = pool.map(one, BATCHES, chunksize=1)
    meta = [m for m, _ in out]
    seqs = [r for _, r in out]
    offs = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum([len(s) for s in seqs], out=offs[1:])
    np.savez_compressed(HERE / "c2_sweep.npz", reqs=np.concatenate(seqs),
                        offsets=offs)
    (HERE / "c2_sweep_golden.json").write_text(json.dumps(
        {"capture": "tools/capture_models.py gpt2 --batch B --seq 128 --iters 3 "
                    "(torch 2.11 CPU profiler, capture.py:79-85 flags)",
         "iterations": 2, "traces": meta}, indent=0) + "\n")
    for m in meta:
        print(m["batch"], m["n_events"], m["n_requests"], m["peak_reserved"],
              f"{m['reference_e2e_s']:.2f}s")


if __name__ == "__main__":
    main()
