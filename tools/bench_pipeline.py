"""Time the estimator pipeline stages on C5-style traces.

    python tools/bench_pipeline.py --leaves 6000 60000 300000

Per size: events, analyze (host tree + pm_link), build_sequence
(pm_orchestrate), replay, with events/s; optional --check runs the CPU
oracle on the same trace and compares the request sequence.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, nargs="+", default=[6000])
    ap.add_argument("--iterations", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--sweep", type=int, default=0,
                    help="also: N event-level traces (leaves 200 k, k = 1..N) "
                         "estimated in one estimate_many call vs a loop of "
                         "per-trace estimate_with_details")
    ap.add_argument("--file", action="store_true",
                    help="also time the user path: write the trace as chrome "
                         "JSON, then parse_trace + estimate from the file")
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.estimator import replay_sequence
    torch.cuda.init()
    # warm the libraries / CUDA context on a tiny trace
    b0 = synth_events.generate(50, args.iterations)
    replay_sequence(api.build_sequence(api.analyze(b0), args.iterations),
                    api.AllocatorConfig())
    if args.sweep:
        bs = [synth_events.generate(200 * k, args.iterations, seed=k)
              for k in range(1, args.sweep + 1)]
        est = api.PeakMemoryEstimator(iterations=args.iterations)
        est.estimate_many(bs[:2])
        t0 = time.perf_counter()
        many = est.estimate_many(bs)
        t1 = time.perf_counter()
        loop = [est.estimate_with_details(b, _timeline=False)[0] for b in bs]
        t2 = time.perf_counter()
        print(json.dumps({
            "sweep_traces": len(bs), "events": sum(len(b) for b in bs),
            "requests": sum(r.sequence_length for r in many),
            "estimate_many_s": t1 - t0, "per_trace_loop_s": t2 - t1,
            "reports_equal": all(a.canonical_json() == b.canonical_json()
                                 for a, b in zip(many, loop))}), flush=True)
    for leaves in args.leaves:
        t0 = time.perf_counter()
        b = synth_events.generate(leaves, args.iterations)
        t_gen = time.perf_counter() - t0
        # warm-up at this size (the device pools grow on the first call)
        tw = time.perf_counter()
        api.build_sequence(api.analyze(b), args.iterations)
        torch.cuda.synchronize()
        t_cold = time.perf_counter() - tw
        t1 = time.perf_counter()
        a = api.analyze(b)
        t2 = time.perf_counter()
        seq = api.build_sequence(a, args.iterations)
        t3 = time.perf_counter()
        res = replay_sequence(seq, api.AllocatorConfig(), timeline=False)
        t4 = time.perf_counter()
        n = len(b)
        # the batched, device-resident path (pm_pipeline_batch) on the same
        # trace: analyze + build_sequence in one call
        from paper_2504_03887_b200.batch import build_sequences
        build_sequences([b], args.iterations)  # warm (pool growth at this size)
        t5 = time.perf_counter()
        sb = build_sequences([b], args.iterations)
        torch.cuda.synchronize()
        t6 = time.perf_counter()
        batch_equal = bool((sb.packed(0) == seq.packed).all())
        t7 = time.perf_counter()
        rep_b = api.PeakMemoryEstimator(iterations=args.iterations).estimate_many([b])[0]
        t8 = time.perf_counter()
        line = {"leaves": leaves, "events": n, "requests": len(seq.packed),
                "batch_analyze_build_s": t6 - t5, "batch_equal": batch_equal,
                "estimate_many_s": t8 - t7,
                "estimate_many_peak_equal": rep_b.reserved_peak == res.peak_reserved,
                "gen_s": t_gen, "cold_analyze_build_s": t_cold, "analyze_s": t2 - t1,
                "build_sequence_s": t3 - t2, "replay_s": t4 - t3,
                "pipeline_events_per_s": n / (t4 - t1),
                "peak_reserved": res.peak_reserved}
        if args.check:
            from oracle import pipeline as op
            recs = b.to_json_dict()["traceEvents"]
            side = {"param_sizes": list(b.metadata.param_sizes),
                    "batch_bytes": list(b.metadata.batch_bytes)}
            tc = time.perf_counter()
            want = op.build_sequence(op.normalize(recs), side, args.iterations)
            line["oracle_s"] = time.perf_counter() - tc
            line["oracle_equal"] = want == [(r.kind.value, r.block_id, r.size,
                                             r.virtual_ts) for r in seq.requests]
        if args.file:
            import tempfile
            from paper_2504_03887_b200.trace import parse_trace
            with tempfile.TemporaryDirectory() as d:
                path = Path(d) / "c5.trace.json"
                # laid out like a profiler's chrome trace: one record per
                # indented block (the torch profiler writes "\n  {" blocks)
                path.write_text(json.dumps(b.to_json_dict(), indent=2))
                line["file_mb"] = path.stat().st_size / 1e6
                tf = time.perf_counter()
                pb = parse_trace(path, b.metadata)
                tg = time.perf_counter()
                est = api.PeakMemoryEstimator(iterations=args.iterations)
                rep = est.estimate(pb)
                th = time.perf_counter()
            line.update({"parse_s": tg - tf, "estimate_s": th - tg,
                         "file_to_report_s": th - tf,
                         "file_peak_equal": rep.reserved_peak == res.peak_reserved})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
