"""BASELINE configs[1] / SURVEY §8d C2 end to end: 64 GPT-2 small training
traces (batch 1..64, seq 128) -> 64 estimate reports, engine vs reference on
the SAME files.

    python tools/bench_c2_e2e.py [--caps DIR] [--capture] [--jobs 4]

--capture runs tools/capture_models.py for every missing batch size (CPU
profiler, capture.py:79-85 flags; `--jobs` captures at a time, 4 threads
each).  Then, for the 64 files:

  reference  the reference package (baseline/_ref) parse_trace +
             PeakMemoryEstimator.estimate per file, one process per file
             (all host cores), and its serial per-file time;
  engine     (1) per file: parse_trace + estimate (a loop);
             (2) batched: the 64 files parsed on host threads, then ONE
             estimate_many (one pm_pipeline_batch + one replay batch).
Reports must be byte-identical to the reference's.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
BATCHES = list(range(1, 65))


def _name(b):
    return f"gpt2_bs{b}_s128"


def capture(caps: Path, jobs: int):
    todo = [b for b in BATCHES if not (caps / _name(b) / "trace.json").exists()]
    env = dict(os.environ, OMP_NUM_THREADS="4")
    running = []
    t0 = time.perf_counter()
    # largest first so the long captures start early
    for b in sorted(todo, reverse=True):
        while len(running) >= jobs:
            running = [p for p in running if p.poll() is None]
            time.sleep(0.2)
        running.append(subprocess.Popen(
            [sys.executable, str(REPO / "tools" / "capture_models.py"), "gpt2",
             "--batch", str(b), "--seq", "128", "--iters", "3"],
            env=env, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL))
    for p in running:
        p.wait()
    return len(todo), time.perf_counter() - t0


def _ref_one(path_pair):
    trace, side = path_pair
    sys.path.insert(0, str(REPO / "baseline" / "_ref"))
    import logging
    logging.disable(logging.WARNING)
    from peakmem import PeakMemoryEstimator, load_sidecar, parse_trace
    t0 = time.perf_counter()
    rep = PeakMemoryEstimator().estimate(
        parse_trace(str(trace), sidecar=load_sidecar(str(side))))
    return rep.canonical_json(), time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--caps", default=str(REPO / "data" / "captures"))
    ap.add_argument("--capture", action="store_true")
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--profile", action="store_true",
                    help="cProfile of the batched parse + estimate_many to stderr")
    ap.add_argument("--no-reference", action="store_true")
    args = ap.parse_args()
    caps = Path(args.caps)
    out = {"config": "C2: GPT-2 small (124M) training traces, batch 1..64 x seq 128, "
                     "AdamW, iterations=2: 64 files -> 64 reports"}
    if args.capture:
        n, dt = capture(caps, args.jobs)
        out["captured"] = {"traces": n, "seconds": dt}
    files = [(caps / _name(b) / "trace.json", caps / _name(b) / "sidecar.json")
             for b in BATCHES]
    missing = [str(t) for t, _ in files if not t.exists()]
    if missing:
        sys.exit(f"missing captures: {missing[:3]} ... (use --capture)")
    out["json_mb"] = round(sum(t.stat().st_size for t, _ in files) / 1e6, 1)

    # reference, one process per file
    ctx = mp.get_context("fork")
    procs = len(os.sched_getaffinity(0))
    if args.no_reference:
        ref, ref_wall = [(None, float("nan"))] * len(files), float("nan")
    else:
        t0 = time.perf_counter()
        with ctx.Pool(procs) as pool:
            ref = pool.map(_ref_one, files, chunksize=1)
        ref_wall = time.perf_counter() - t0
    ref_reports = [r for r, _ in ref]
    out["reference"] = {"wall_s": ref_wall, "processes": procs,
                        "serial_s": sum(t for _, t in ref)}

    import logging
    logging.disable(logging.WARNING)
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    est = eng.PeakMemoryEstimator()

    def parse(pair):
        return eng.parse_trace(pair[0], sidecar=eng.load_sidecar(pair[1]))

    # warm-up: CUDA context, libraries, pools
    est.estimate_many([parse(files[0]), parse(files[1])])
    torch.cuda.synchronize()
    # (1) a loop over files
    t0 = time.perf_counter()
    loop = [est.estimate(parse(f)).canonical_json() for f in files]
    t_loop = time.perf_counter() - t0
    # (2) batched: parse on host threads, one estimate_many
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=8) as pool:
        bundles = list(pool.map(parse, files))
    t1 = time.perf_counter()
    many = [r.canonical_json() for r in est.estimate_many(bundles)]
    t2 = time.perf_counter()
    out["engine_loop"] = {"s": t_loop,
                          "reports_identical": f"{sum(a == b for a, b in zip(loop, ref_reports))}/64"}
    out["engine_batched"] = {"s": t2 - t0, "parse_s": t1 - t0, "estimate_many_s": t2 - t1,
                             "reports_identical": f"{sum(a == b for a, b in zip(many, ref_reports))}/64"}
    out["speedup_batched_vs_reference_wall"] = ref_wall / (t2 - t0)
    out["speedup_batched_vs_reference_serial"] = out["reference"]["serial_s"] / (t2 - t0)
    print(json.dumps(out), flush=True)
    if args.profile:
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        with ThreadPoolExecutor(max_workers=8) as pool:
            bundles = list(pool.map(parse, files))
        est.estimate_many(bundles)
        pr.disable()
        pstats.Stats(pr, stream=sys.stderr).sort_stats("cumtime").print_stats(40)


if __name__ == "__main__":
    main()
