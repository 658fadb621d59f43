"""End to end, one captured trace -> report (BASELINE configs C1 / C2): the
reference package (baseline/_ref, pure Python, CPU) vs this engine, same
host, same files; the two reports must be byte-identical.

    python tools/bench_estimate.py [--repeat 5]

Prints one JSON line per capture: median seconds of
`PeakMemoryEstimator().estimate(parse_trace(file, sidecar=load_sidecar(...)))`
for each side (parse included, file already decompressed on local disk).
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

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
CAPTURES = ("resnet18_bs32_224", "gpt2_bs8_s128")


def timed(fn, repeat):
    out, times = None, []
    for _ in range(repeat):
        t0 = time.perf_counter()
        out = fn()
        times.append(time.perf_counter() - t0)
    return out, statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeat", type=int, default=5)
    args = ap.parse_args()
    import logging
    logging.disable(logging.WARNING)
    import torch  # noqa: F401  (CUDA context for the engine)
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    ref_root = REPO / "baseline" / "_ref"
    if not (ref_root / "peakmem").exists():
        ref_root = Path("/root/reference/pkg/src")
    sys.path.insert(0, str(ref_root))
    import peakmem as ref

    golden = REPO / "tests" / "golden" / "traces"
    tmp = Path(tempfile.mkdtemp())
    # warm the engine (CUDA context, libraries) on the small fixture
    small = tmp / "tiny.json"
    small.write_bytes(gzip.open(golden / "tiny_mlp_adam.trace.json.gz").read())
    eng.PeakMemoryEstimator().estimate(
        eng.parse_trace(small, sidecar=eng.load_sidecar(golden / "tiny_mlp_adam.sidecar.json")))
    for name in CAPTURES:
        trace = tmp / f"{name}.json"
        trace.write_bytes(gzip.open(golden / f"{name}.trace.json.gz").read())
        side = golden / f"{name}.sidecar.json"
        r_ref, t_ref = timed(lambda: ref.PeakMemoryEstimator().estimate(
            ref.parse_trace(trace, sidecar=ref.load_sidecar(side))), args.repeat)
        r_eng, t_eng = timed(lambda: eng.PeakMemoryEstimator().estimate(
            eng.parse_trace(trace, sidecar=eng.load_sidecar(side))), args.repeat)
        print(json.dumps({
            "capture": name, "trace_mb": round(trace.stat().st_size / 1e6, 1),
            "reference_s": t_ref, "engine_s": t_eng, "speedup": t_ref / t_eng,
            "reports_identical": r_ref.canonical_json() == r_eng.canonical_json(),
            "predicted_peak": r_eng.predicted_peak if hasattr(r_eng, "predicted_peak") else None,
        }), flush=True)


if __name__ == "__main__":
    main()
