"""Benchmark: replayed allocator events/s for batched traces on B200.

Metric (BASELINE.json): "replayed allocator events/sec (batched traces,
1/2/4/8 B200); bit-exact peak bytes".  Workload:
10^4 synthetic Llama-style request traces of ~1e5 requests each (~1e9
requests, 16 GB packed), default AllocatorConfig, unbounded capacity.  Traces
are independent, so with N GPUs every rank replays its own 10^4-trace C3
sweep (traces r*10^4 .. r*10^4+9999, distinct seeds) with no collective on
the data path: weak scaling, `value` = all ranks' requests / the slowest
rank's time.  `--strong` instead shards ONE 10^4-trace sweep over the ranks
by greedy LPT on length.

  value   device-resident: packed requests already in HBM, one step = one
          pm_replay_batch over the rank's shard, timed with CUDA events on
          the launching stream, max over ranks.
  e2e     the same step through the C ABI with HOST buffers
          (pm_replay_host_wire: pinned host requests in the 8-byte wire
          format -> H2D -> replay -> D2H of the per-trace results),
          wall-clock around the synchronous call.
  roofline  HBM: 16 B of packed request read per replayed event
           / the replay launch's CUDA-event duration, against
          MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the C oracle port of the reference allocator
          (oracle/replay_oracle.c) on every 10th trace of rank 0's shard, all
          host threads; its per-trace results double as a parity check.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port; the reference itself is Python and does not travel to the GPU
box) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

BYTES_PER_EVENT = 16  # algorithmic: one packed request read
METRIC = "replayed allocator events/sec (batched traces, 1/2/4/8 B200); bit-exact peak bytes"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--traces", type=int, default=10_000,
                    help="traces per rank (weak scaling) or in total (--strong)")
    ap.add_argument("--strong", action="store_true",
                    help="shard one fixed sweep of --traces traces over the ranks "
                         "(default: every rank replays its own --traces traces)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-sample-stride", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def read_peak():
    p = REPO / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(reqs, offsets, cfg, stride: int, gpu_results=None):
    """Oracle port on every `stride`-th trace, all host threads."""
    from oracle import replay as oracle
    idx = np.arange(0, len(offsets) - 1, stride)
    parts = [reqs[offsets[i]:offsets[i + 1]] for i in idx]
    sub_offs = np.zeros(len(idx) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=sub_offs[1:])
    sub = np.concatenate(parts)
    threads = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    res, _ = oracle.replay_batch(sub, sub_offs, cfg, n_threads=threads)
    dt = time.perf_counter() - t0
    events = int(res["n_events_replayed"].sum())
    # SURVEY §8d also asks for a 1-core figure: every 10th trace of the sample
    k1 = max(1, len(idx) // 10)
    t1 = time.perf_counter()
    r1, _ = oracle.replay_batch(sub[:sub_offs[k1]], sub_offs[:k1 + 1], cfg,
                                n_threads=1)
    dt1 = time.perf_counter() - t1
    ev1 = int(r1["n_events_replayed"].sum())
    out = {"value": events / dt, "unit": "events/s", "cores": threads,
           "kind": "port",
           "sample": f"every {stride}th trace of the rank-0 shard: "
                     f"{len(idx)} traces, {events} requests, {dt:.2f} s wall",
           "value_1core": ev1 / dt1,
           "sample_1core": f"first {k1} traces of that sample, {ev1} requests, "
                           f"{dt1:.2f} s on 1 thread"}
    parity = None
    if gpu_results is not None:
        mism = int((gpu_results[idx] != res).sum())
        parity = {"checked_traces": int(len(idx)), "mismatches": mism,
                  "fields": "all pm_result_t fields (peaks, finals, status, "
                            "stop index, segment counts, pool high-water)"}
    return out, parity


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import __graft_entry__

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # rank 0 (re)builds if a source is newer than its library; the others
    # load the libraries only after it is done
    if rank == 0:
        __graft_entry__.build()
    if dist:
        dist.barrier()
    from paper_2504_03887_b200 import _native, synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # ---- workload ----------------------------------------------------------
    # weak scaling (default): rank r replays its own C3 sweep, traces
    # r*T .. r*T+T-1 (seeds 1_000_003 + i); --strong: the ranks share one
    # sweep of T traces by greedy LPT on length.  No collective on the data
    # path either way.
    from paper_2504_03887_b200.synth import _load
    lib = _load()
    n_all = args.traces if args.strong else args.traces * world
    counts = np.zeros(n_all, dtype=np.int64)
    lib.pm_synth_counts(0, n_all, counts.ctypes.data,
                        len(os.sched_getaffinity(0)))
    from paper_2504_03887_b200.shard import lpt_shards
    if args.strong:
        mine = lpt_shards(counts, world)[rank]
    else:
        mine = np.arange(rank * args.traces, (rank + 1) * args.traces)
    # generate the rank's traces contiguously
    offs = np.zeros(len(mine) + 1, dtype=np.int64)
    np.cumsum(counts[mine], out=offs[1:])
    total = int(offs[-1])
    # pageable: these records are copied to the device once, outside the
    # timed regions (only the e2e input, the wire words below, is pinned)
    reqs = np.empty(total, dtype=_native.REQ_DTYPE)
    # traces of the shard are not contiguous in index space: fill one by one
    # range at a time (consecutive runs of trace ids)
    runs = np.split(np.arange(len(mine)), np.nonzero(np.diff(mine) != 1)[0] + 1)
    threads = len(os.sched_getaffinity(0))
    for run in runs:
        first = int(mine[run[0]])
        sub_offs = (offs[run[0]:run[-1] + 2] - offs[run[0]]).copy()
        lib.pm_synth_fill(first, len(run), sub_offs.ctypes.data,
                          reqs[offs[run[0]]:].ctypes.data, threads)
    cfg = cfg_record(AllocatorConfig())

    batch = DeviceBatch(reqs, offs, cfg, device=local)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        batch.launch(stream)
    torch.cuda.synchronize(dev)
    results = batch.results()
    bad = np.nonzero(results["status"] != 0)[0]
    if len(bad):
        raise RuntimeError(f"{len(bad)} traces ended with status "
                           f"{np.unique(results['status'][bad])}")
    events_per_step = int(results["n_events_replayed"].sum())

    # ---- timed region: K device-resident steps -----------------------------
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record(stream)
        for k in range(args.steps):
            starts[k].record(stream)
            batch.launch(stream)
            ends[k].record(stream)
        t_all1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    elapsed_ms = t_all0.elapsed_time(t_all1)
    launch_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    stats = torch.tensor([elapsed_ms, float(events_per_step)], dtype=torch.float64,
                         device=dev)
    if dist:
        t = stats[:1].clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ev = stats[1:].clone()
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
        max_ms, all_events = float(t.item()), float(ev.item())
    else:
        max_ms, all_events = elapsed_ms, float(events_per_step)
    value = all_events * args.steps / (max_ms / 1e3)

    # ---- e2e: host buffers through the C ABI ------------------------------
    # The host packs its requests once into the engine's 8-byte wire format
    # (pm_wire_pack, like pack_trace builds pm_req_t; outside the timed
    # region); each timed step is pm_replay_host_wire: H2D of the words
    # (pinned), replay, D2H of the per-trace results.
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    whost = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
    words = _native.wire_pack(reqs, offs, out=whost.numpy().view(np.uint64))
    if words is None:
        raise RuntimeError("C3 requests must have a wire encoding")
    _native.replay_host_wire(words, offs, cfg, None, False)  # pool warm-up
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res_host, _ = _native.replay_host_wire(words, offs, cfg, None, False)
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = all_events * e2e_steps / float(e2e_t.item())
    if (res_host != results).any():
        raise RuntimeError("host-buffer path disagrees with device-resident path")

    # ---- roofline of the replay launch -------------------------------------
    mean_launch_s = statistics.mean(launch_ms) / 1e3
    achieved = events_per_step * BYTES_PER_EVENT / mean_launch_s / 1e9
    peak, peak_kind = read_peak()
    traffic = None
    issue = None
    prof = REPO / "profiles" / "replay_ncu_summary.json"
    if prof.exists():
        summ = json.loads(prof.read_text())
        # same unit as `achieved`: DRAM bytes per launch / launch time
        traffic = summ["dram_bytes_per_event"] * events_per_step / mean_launch_s / 1e9
        # the real bound is issue -- SMs x 4 schedulers x clock /
        # warp-instructions per event (ncu-measured, profiles/)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        issue = {"warp_instructions_per_event": summ["warp_instructions_per_event"],
                 "sms": sms, "schedulers_per_sm": 4}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    cpu, parity = (None, None)
    if not args.no_cpu_baseline and world >= 1:
        cpu, parity = cpu_baseline(reqs, offs, cfg, args.cpu_sample_stride,
                                   results)
        if parity and parity["mismatches"]:
            raise RuntimeError(f"parity failure vs oracle: {parity}")

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "events/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded Llama-style request traces, SURVEY §8d C3)",
        "config": {
            "workload": ("C3: one sweep of 10^4 synthetic Llama-style training "
                         "traces (~1e5 requests each) sharded LPT over the GPUs"
                         if args.strong else
                         "C3: 10^4 synthetic Llama-style training traces (~1e5 "
                         "requests each) per GPU, distinct seeds per rank"),
            "n_traces": args.traces if args.strong else args.traces * world,
            "requests_total_all_ranks": int(all_events),
            "requests_rank0": events_per_step,
            "allocator": "AllocatorConfig() defaults, device_capacity None",
            "l2": "inputs larger than L2 (16 B x ~1e9 requests >> 126 MB)",
            "parallelism": f"independent traces over {world} GPU(s), no collective "
                           "on the data path (NCCL only for the barrier and the "
                           "max-over-ranks time)",
        },
        "e2e": {"value": e2e_value, "unit": "events/s",
                "h2d_bytes_per_step": int(words.nbytes + offs.nbytes + cfg.nbytes),
                "d2h_bytes_per_step": int(res_host.nbytes),
                "steps": e2e_steps,
                "api": "pm_replay_host_wire (C ABI, pinned host buffers, 8-byte "
                       "wire words packed by pm_wire_pack outside the timed region)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "traffic": traffic,
                     "traffic_note": "GB/s: DRAM read+write bytes per event from the ncu "
                                     "--set full capture (profiles/replay_ncu_summary.json) "
                                     "x events per launch / launch time",
                     "kernel": "replay_narrow_kernel<24> (main pass, 100 % of GPU time in profiles/r01_v8_bench_launches.csv; the six retry-pass kernels ride in the same timed launch)",
                     "algorithmic_bytes_per_event": BYTES_PER_EVENT},
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clocks.summary(),
        "issue_bound": issue,
        "gpu_launches": 7 * args.steps,  # main pass + 2 narrow + 4 wide retry passes per pm_replay_batch
    }
    if issue is not None:
        mhz = line["clocks"]["sm_mhz"] or 1965.0
        ceiling = issue["sms"] * 4 * mhz * 1e6 / issue["warp_instructions_per_event"]
        issue.update({"clock_mhz": mhz, "ceiling_events_per_s": ceiling,
                      "frac": value / (ceiling * world),
                      "source": "profiles/replay_ncu_summary.json (ncu --set full "
                                "of the replay kernel: instructions, DRAM bytes)"})
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """Reference arm: the reference algorithm's CPU implementation (the
    oracle port of allocator.py) on the box's host cores, rank 0 only."""
    if rank != 0:
        return
    import __graft_entry__
    __graft_entry__.build()
    from oracle import replay as oracle
    from paper_2504_03887_b200 import synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    stride = args.cpu_sample_stride
    idx = np.arange(0, args.traces, stride)
    threads = len(os.sched_getaffinity(0))
    parts, lens = [], []
    for i in idx:
        r, o = synth.generate(1, first=int(i), n_threads=1)
        parts.append(r.copy())
        lens.append(len(r))
    offs = np.zeros(len(idx) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    reqs = np.concatenate(parts)
    cfg = cfg_record(AllocatorConfig())
    for _ in range(min(args.warmup, 1)):
        oracle.replay_batch(reqs[:offs[min(8, len(idx))]],
                            offs[:min(8, len(idx)) + 1], cfg, n_threads=threads)
    times, events = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res, _ = oracle.replay_batch(reqs, offs, cfg, n_threads=threads)
        times.append(time.perf_counter() - t0)
        events = int(res["n_events_replayed"].sum())
    value = events * len(times) / sum(times)
    sample = (f"every {stride}th trace of the 10^4-trace C3 sweep: {len(idx)} "
              f"traces, {events} requests per step")
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded Llama-style request traces, SURVEY §8d C3)",
        "config": {"workload": "C3: 10^4 synthetic Llama-style training traces, "
                               "~1e5 requests each (bounded CPU sample)",
                   "n_traces": args.traces,
                   "allocator": "AllocatorConfig() defaults, device_capacity None"},
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "implementation": "oracle/replay_oracle.c: C restatement of "
                          "peakmem.allocator (the reference is pure Python; "
                          "its own throughput is reported beside it)",
    }
    py = reference_python_rate(reqs, offs, threads)
    if py is not None:
        line["reference_python"] = py
    print(json.dumps(line))


def _py_replay_worker(args):
    """One trace through the reference's own replay (baseline/_ref)."""
    root, recs = args
    sys.path.insert(0, root)
    import time as _t
    from peakmem.allocator import AllocatorConfig as RC, replay as rreplay
    t0 = _t.perf_counter()
    rreplay(recs, RC())
    return len(recs), _t.perf_counter() - t0


def reference_python_rate(reqs, offs, threads, n_traces=16):
    """The reference's own Python replay (peakmem.allocator.replay from the
    pip-installed baseline/_ref) on the first few sampled traces, one
    process per trace over all host cores: context for the C port above."""
    root = REPO / "baseline" / "_ref"
    if not (root / "peakmem").exists():
        return None
    import multiprocessing as mp
    jobs = []
    for t in range(min(n_traces, len(offs) - 1)):
        r = reqs[offs[t]:offs[t + 1]]
        kinds = ("alloc", "free")
        recs = [{"seq_no": i, "kind": kinds[int(k) & 3], "block_id": int(h),
                 "size": int(sz)} for i, (sz, h, k) in
                enumerate(zip(r["size"].tolist(), r["handle"].tolist(),
                              r["kind_stream"].tolist()))]
        jobs.append((str(root), recs))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(threads) as pool:
        out = pool.map(_py_replay_worker, jobs)
    wall = time.perf_counter() - t0
    events = sum(n for n, _ in out)
    per_core = events / sum(dt for _, dt in out)
    return {"value": events / wall, "unit": "events/s", "cores": threads,
            "per_core": per_core,
            "sample": f"{len(jobs)} C3 traces ({events} requests), "
                      "peakmem.allocator.replay from baseline/_ref, one process per trace"}


if __name__ == "__main__":
    main()
