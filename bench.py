"""Benchmark: replayed allocator events/s for batched traces on B200.

Metric (BASELINE.json): "replayed allocator events/sec (batched traces,
1/2/4/8 B200); bit-exact peak bytes".  Workload (SURVEY.md §8d, config C3,
BASELINE configs[2]): ONE sweep of 10^4 synthetic Llama-style request traces
of ~1e5 requests each (~1e9 requests, 16 GB packed; trace i drawn from numpy
PCG64(1_000_003 + i), oracle/c3gen.py == workloads/c3gen.c), default
AllocatorConfig, unbounded capacity, sharded over the GPUs by greedy LPT on
length with no collective on the data path (strong scaling).  `--weak` gives
every rank its own 10^4-trace sweep instead.

  value   device-resident: the rank's packed requests already in HBM, one
          step = one pm_replay_batch over its shard, CUDA events on the
          launching stream, max over ranks; value = all ranks' requests /
          that time.
  e2e     the same step through the C ABI with HOST buffers: the workload
          in the engine's 8-byte wire format as the generator emits it
          (packed once at generation time, outside the timed region),
          pm_replay_host_wire reading it over PCIe in place, + D2H of the
          per-trace results.  Beside it: `e2e_req16` = pm_replay_host on
          pinned 16 B pm_req_t records (the documented ABI record, read in
          place); `e2e_wire` = pm_wire_pack (host threads) INSIDE the timed
          region + pm_replay_host_wire.
  roofline  HBM: 16 B of packed request read per replayed event
           / the replay launch's CUDA-event duration, against
          MEASURED_PEAKS.json hbm_gbs; `issue_bound` beside it.
  cpu_baseline  (rank 0, N=1) the C port of the reference allocator
          (oracle/replay_oracle.c) on every 10th trace of the shard, all host
          threads; its results double as a parity check.
  parity.reference_*  the REFERENCE itself (peakmem.allocator.AllocatorState
          from baseline/_ref, one process per trace) on 16 traces of rank 0's
          shard, every result field compared with the GPU's.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port -- the reference is Python; its own rate is printed beside it) on
the same workload: each step replays a different 1/20 of the sweep (step s:
traces i with i % 20 == s % 20), so 20 timed steps cover every trace once.
It loads only oracle/lib/liboracle_replay.so (replay + the same C3
generator), never the engine.  Under torchrun rank 0 alone runs it.

`--gpus N` without torchrun's WORLD_SIZE re-launches itself under
torch.distributed.run with N ranks.  `--dry-run` runs the multi-rank host
path on CPU (gloo; each rank replays its shard with the oracle) to prove the
spawn / shard / gather / max-reduce plumbing without a GPU; it prints
`"dry_run": true` and is never a bench value.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
RESIDENT_WARPS_PER_SM = 24  # replay_narrow_kernel<24>, one CTA per SM
REF_STRIDE = 20             # reference arm: 1/20 of the sweep per step


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--traces", type=int, default=10_000,
                    help="traces in the sweep (strong) or per rank (--weak)")
    ap.add_argument("--weak", action="store_true",
                    help="every rank replays its own --traces traces")
    ap.add_argument("--strong", action="store_true",
                    help="(default) shard one sweep of --traces traces")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-sample-stride", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shared-device", action="store_true",
                    help="plumbing check on a one-GPU machine: every rank uses "
                         "cuda:0 and the gloo backend (timings are not a "
                         "scaling measurement)")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the C2 / C4 / C5 measurements beside the C3 line")
    ap.add_argument("--ref-check-traces", type=int, default=16)
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo plumbing check (oracle replay); not a bench value")
    return ap.parse_args(argv)


def sweep_ids(args, world: int) -> np.ndarray:
    n = args.traces * world if args.weak else args.traces
    return np.arange(n, dtype=np.int32)


def workload_config(args, world: int) -> dict:
    """The `config` both arms print (identical dicts)."""
    n = args.traces * world if args.weak else args.traces
    if args.weak:
        wl = (f"C3: {args.traces} synthetic Llama-style training traces (~1e5 "
              "requests each) per GPU, distinct traces per rank")
    else:
        wl = (f"C3: one sweep of {args.traces} synthetic Llama-style training "
              "traces (~1e5 requests each), sharded LPT over the GPUs")
    return {
        "workload": wl,
        "n_traces": n,
        "generator": "numpy Generator(PCG64(1_000_003 + i)) per trace "
                     "(oracle/c3gen.py spec; workloads/c3gen.c)",
        "allocator": "AllocatorConfig() defaults, device_capacity None",
        "l2": "inputs larger than L2 (16 B x ~1e9 requests >> 126 MB)",
        "parallelism": f"independent traces over {world} GPU(s), no collective "
                       "on the data path (NCCL only for the barrier, the "
                       "max-over-ranks time and the result gather)",
    }


def read_peak():
    p = REPO / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_info() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "affinity_cores": len(os.sched_getaffinity(0))}


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


# ---- the reference itself as a checker (baseline/_ref) ----------------------

def _ref_root() -> Path | None:
    for cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "peakmem" / "allocator.py").exists():
            return cand
    return None


def _ref_worker(job):
    """One packed trace through the reference's AllocatorState, driven as
    replay() drives it (allocator.py:360-393), reading segment counts and
    the free-pool size too.  Returns (result fields, requests, seconds)."""
    root, size, handle, ks = job
    if root not in sys.path:
        sys.path.insert(0, root)
    from peakmem.allocator import AllocatorConfig, AllocatorState
    from peakmem.errors import OutOfMemory
    t0 = time.perf_counter()
    st = AllocatorState(AllocatorConfig())
    nseg_peak = max_pool = 0
    status, stop, n = 0, -1, 0
    for i, (sz, h, k) in enumerate(zip(size, handle, ks)):
        try:
            if k & 3 == 0:
                st.allocate(h, sz, k >> 2)
            else:
                st.free(h)
        except OutOfMemory:
            status, stop = 1, i
            nseg_peak = max(nseg_peak, len(st.segments))
            n += 1
            break
        st.step(i)
        n += 1
        nseg_peak = max(nseg_peak, len(st.segments))
        max_pool = max(max_pool, len(st.free_pool))
    out = (st.peak_reserved, st.peak_allocated, st.reserved_bytes,
           st.allocated_bytes, stop, n, status, len(st.segments), nseg_peak,
           max_pool)
    return out, len(size), time.perf_counter() - t0


def reference_replay(reqs, offs, idx, threads):
    """The reference's own replay on traces `idx` of a packed batch, one
    process per trace.  Returns (RESULT-shaped array, wall s, per-core rate)
    or None when the reference is not importable."""
    root = _ref_root()
    if root is None or len(idx) == 0:
        return None
    import multiprocessing as mp
    jobs = []
    for t in idx:
        r = reqs[offs[t]:offs[t + 1]]
        jobs.append((str(root), r["size"].tolist(), r["handle"].tolist(),
                     r["kind_stream"].tolist()))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(threads, len(jobs))) as pool:
        out = pool.map(_ref_worker, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    from oracle.replay import RESULT_DTYPE
    res = np.zeros(len(idx), dtype=RESULT_DTYPE)
    for k, (vals, _, _) in enumerate(out):
        res[k] = vals
    events = sum(n for _, n, _ in out)
    per_core = events / sum(dt for _, _, dt in out)
    return res, wall, events, per_core


# ---- engine arm ---------------------------------------------------------------

def _relaunch(args) -> int:
    """--gpus N without WORLD_SIZE: N ranks under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def _gather(dist, obj, world):
    if dist is None:
        return [obj]
    parts = [None] * world
    dist.all_gather_object(parts, obj)
    return parts


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", 0))
    if world == 0 and args.gpus > 1:
        sys.exit(_relaunch(args))
    world = max(world, 1)
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.shared_device:
        local = 0
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.dry_run:
        return run_dry(args, rank, world)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.shared_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:  # no-op when the in-tree libraries are up to date
        import __graft_entry__
        __graft_entry__.build()
    if dist:
        dist.barrier()
    from paper_2504_03887_b200 import _native, synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.engine import DeviceBatch
    from paper_2504_03887_b200.shard import lpt_shards
    _native.load_library()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    threads = len(os.sched_getaffinity(0))

    # ---- workload: this rank's shard, generated into pinned memory ---------
    ids = sweep_ids(args, world)
    if args.weak:
        mine = ids[rank * args.traces:(rank + 1) * args.traces]
        lengths = synth.counts(mine, threads)
    else:
        all_len = synth.counts(ids, threads)
        mine = lpt_shards(all_len, world)[rank].astype(np.int32)
        lengths = all_len[mine]
    total = int(lengths.sum())
    pinned = torch.empty(total * 16, dtype=torch.uint8, pin_memory=True)
    reqs, offs = synth.generate_ids(
        mine, threads, out=pinned.numpy().view(_native.REQ_DTYPE),
        lengths=lengths)
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
    # reductions live where the backend can reduce them (gloo: host)
    rdev = torch.device("cpu") if args.shared_device else dev
    if dist:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ev = torch.tensor([float(events_per_step)], dtype=torch.float64, device=rdev)
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
        max_ms, all_events = float(t.item()), float(ev.item())
    else:
        max_ms, all_events = elapsed_ms, float(events_per_step)
    value = all_events * args.steps / (max_ms / 1e3)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    rank_info = {"rank": rank, "traces": int(len(mine)),
                 "requests": events_per_step,
                 "ms_per_step": elapsed_ms / args.steps,
                 "resident_warp_slots": sms * RESIDENT_WARPS_PER_SM,
                 "waves": round(len(mine) / (sms * RESIDENT_WARPS_PER_SM), 3)}

    # ---- e2e: host buffers through the C ABI --------------------------------
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))

    def timed_host(fn):
        fn()  # warm-up (pool mapping)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            out = fn()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=rdev)
        if dist:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return out, all_events * e2e_steps / float(tt.item())

    # (1) pm_replay_host on the pinned 16 B pm_req_t records
    res_host, e2e_value = timed_host(
        lambda: _native.replay_host(reqs, offs, cfg, None, False)[0])
    # (2) the wire path, packing included
    whost = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
    wbuf = whost.numpy().view(np.uint64)

    def wire_step():
        words = _native.wire_pack(reqs, offs, out=wbuf)
        if words is None:
            raise RuntimeError("C3 requests must have a wire encoding")
        return _native.replay_host_wire(words, offs, cfg, None, False)[0]
    res_wire, e2e_wire = timed_host(wire_step)
    # (3) the workload as the generator's 8-byte wire words (packed once at
    # generation time, outside the timed region): pm_replay_host_wire reads
    # them over PCIe in place -- half the bytes of (1)
    words_in = _native.wire_pack(reqs, offs, out=wbuf)
    res_win, e2e_win = timed_host(
        lambda: _native.replay_host_wire(words_in, offs, cfg, None, False)[0])
    if ((res_host != results).any() or (res_wire != results).any()
            or (res_win != results).any()):
        raise RuntimeError("host-buffer paths disagree with device-resident path")

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
        issue = {"warp_instructions_per_event": summ["warp_instructions_per_event"],
                 "sms": sms, "schedulers_per_sm": 4,
                 "smsp_issue_active_pct": summ.get("smsp_issue_active_pct"),
                 "thread_inst_per_warp_inst": summ.get("thread_inst_per_warp_inst")}

    ranks = _gather(dist, rank_info, world)

    # ---- parity: the reference itself, and the oracle port ------------------
    ref_parity = None
    cpu, parity = None, None
    if rank == 0:
        k = min(args.ref_check_traces, len(mine))
        pick = np.linspace(0, len(mine) - 1, k).astype(np.int64) if k else []
        got = reference_replay(reqs, offs, pick, threads)
        if got is not None:
            ref_res, wall, ev, per_core = got
            mism = int((results[pick] != ref_res).sum())
            ref_parity = {"reference_checked_traces": int(k),
                          "reference_mismatches": mism,
                          "reference_checked_requests": int(ev),
                          "reference_trace_ids": [int(mine[i]) for i in pick],
                          "reference": "peakmem.allocator.AllocatorState "
                                       "(baseline/_ref), every pm_result_t field",
                          "reference_python_rate": {
                              "value": ev / wall, "unit": "events/s",
                              "cores": min(threads, int(k)), "per_core": per_core}}
            if mism:
                raise RuntimeError(f"parity failure vs the reference: {ref_parity}")
        if not args.no_cpu_baseline and world == 1:
            cpu, parity = cpu_baseline(reqs, offs, cfg, args.cpu_sample_stride,
                                       results)
            if parity and parity["mismatches"]:
                raise RuntimeError(f"parity failure vs oracle: {parity}")
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    parity = dict(parity or {})
    if ref_parity:
        parity.update(ref_parity)
    h2d16 = int(reqs.nbytes + offs.nbytes + cfg.nbytes)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "events/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded Llama-style request traces, SURVEY §8d C3)",
        "config": workload_config(args, world),
        "requests_per_step": int(all_events),
        "e2e": {"value": e2e_win, "unit": "events/s",
                "h2d_bytes_per_step": int(total * 8 + offs.nbytes + cfg.nbytes),
                "d2h_bytes_per_step": int(res_win.nbytes),
                "steps": e2e_steps,
                "api": "pm_replay_host_wire (C ABI) on the workload generator's "
                       "output in the engine's 8-byte wire format (pinned host "
                       "memory, packed once at generation time, outside the timed "
                       "region; read in place over PCIe) + D2H of the per-trace "
                       "results; one synchronous call timed on the host"},
        "e2e_req16": {"value": e2e_value, "unit": "events/s",
                      "h2d_bytes_per_step": h2d16,
                      "d2h_bytes_per_step": int(res_host.nbytes),
                      "steps": e2e_steps,
                      "api": "pm_replay_host (C ABI): pinned host pm_req_t records "
                             "(16 B, read in place over PCIe), D2H of the per-trace "
                             "results, synchronous call timed on the host"},
        "e2e_wire": {"value": e2e_wire, "unit": "events/s",
                     "h2d_bytes_per_step": int(total * 8 + offs.nbytes + cfg.nbytes),
                     "d2h_bytes_per_step": int(res_wire.nbytes),
                     "steps": e2e_steps,
                     "api": "pm_wire_pack (host threads, inside the timed "
                            "region) + pm_replay_host_wire: 8-byte wire words"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "traffic": traffic,
                     "traffic_note": "GB/s: DRAM read+write bytes per event from the ncu "
                                     "--set full capture (profiles/replay_ncu_summary.json) "
                                     "x events per launch / launch time",
                     "kernel": "replay_narrow_kernel<24> (main pass; the retry-pass "
                               "kernels ride in the same timed pm_replay_batch)",
                     "algorithmic_bytes_per_event": BYTES_PER_EVENT},
        "cpu_baseline": cpu,
        "parity": parity or None,
        "ranks": ranks,
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
    if args.shared_device:
        line["shared_device"] = ("plumbing check: every rank on cuda:0 over gloo; "
                                 "not a scaling measurement")
    if world == 1 and not args.no_other_configs:
        line["other_configs"] = other_configs(dev)
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def other_configs(dev) -> dict:
    """BASELINE.json's other configs, measured in the same run (rank 0, N=1)
    so that they are driver-measured too; each checked for parity.

    c2  64 GPT-2 small sequences (batch sizes 1..64, tests/golden/c2_sweep.npz)
        as ONE device-resident replay batch, median of 20 launches (CUDA
        events); every result field vs the reference's (c2_sweep_golden.json).
    c4  50 traces x 69 allocator configs (tools/bench_c4.py's batch), best
        of 5 with the median beside it (parity: the GPU tests against the
        reference's grid goldens).
    c5  one 10^7-event C5-style event-level trace: the batched device
        pipeline (analyze + build_sequence, pm_pipeline_batch) and the
        single-trace replay of its 4.3e6 requests, wall clock; peak vs the
        per-trace API's sequence replayed by the C oracle is in the tests.
    """
    import torch
    sys.path.insert(0, str(REPO / "tests"))
    from paper_2504_03887_b200 import synth, synth_events
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    from paper_2504_03887_b200.batch import build_sequences
    from paper_2504_03887_b200.engine import DeviceBatch
    out = {}
    stream = torch.cuda.current_stream(dev)

    def device_ms(batch, reps):
        batch.launch(stream)
        torch.cuda.synchronize(dev)
        ms = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            batch.launch(stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(e0.elapsed_time(e1))
        return ms

    # C2
    z = np.load(REPO / "tests" / "golden" / "c2_sweep.npz")
    gold = json.loads((REPO / "tests" / "golden" / "c2_sweep_golden.json").read_text())
    b = DeviceBatch(z["reqs"], z["offsets"], cfg_record(AllocatorConfig()), device=dev.index)
    ms = statistics.median(device_ms(b, 20))
    res = b.results()
    fields = ("peak_reserved", "peak_allocated", "final_reserved", "final_allocated",
              "n_segments_final", "n_segments_peak")
    mism = sum(int(res[i][f]) != g[f] for i, g in enumerate(gold["traces"]) for f in fields)
    n2 = int(z["offsets"][-1])
    out["c2"] = {"workload": "64 GPT-2 small training sequences (batch 1..64, seq 128, "
                             "AdamW, 2 iterations) as one replay batch",
                 "requests": n2, "ms": ms, "value": n2 / (ms / 1e3), "unit": "events/s",
                 "reference_mismatches": mism, "timing": "CUDA events, median of 20"}
    # C4
    from c4_cases import c4_batch, c4_configs
    zc = np.load(REPO / "tests" / "golden" / "c2_sequences.npz")
    r3, o3 = synth.generate(42, first=9000)
    reqs = np.concatenate([zc["reqs"], r3])
    offs = np.concatenate([zc["offsets"], o3[1:] + zc["offsets"][-1]])
    big, boffs, rec, cfg_of = c4_batch(reqs, offs, c4_configs())
    b = DeviceBatch(big, boffs, rec, cfg_of, device=dev.index)
    ms_all = device_ms(b, 5)
    ms = min(ms_all)
    res = b.results()
    ev4 = int(res["n_events_replayed"].sum())
    out["c4"] = {"workload": "50 traces (8 GPT-2 sequences + 42 C3) x 69 allocator "
                             "configs = 3450 replays, one batch",
                 "requests": ev4, "ms": ms, "value": ev4 / (ms / 1e3), "unit": "events/s",
                 "ms_median": statistics.median(ms_all),
                 "ms_all": [round(x, 2) for x in ms_all],
                 "retry_passes": b.tier_counts(),
                 "statuses": sorted(set(res["status"].tolist())),
                 "parity": "tests/test_c4_sweep.py, tests/test_config_goldens.py "
                           "(the reference's goldens on the grid)",
                 "timing": "CUDA events, best of 5 (median and every launch beside it: the "
                           "overflowing replays' hand-off timing varies launch to launch)"}
    # C1 (and one C2 batch size): a captured trace file -> report, end to end
    import gzip
    import tempfile
    import paper_2504_03887_b200 as eng
    gold = json.loads((REPO / "tests" / "golden" / "captures_golden.json").read_text())
    tdir = Path(tempfile.mkdtemp())
    for key, name in (("c1", "resnet18_bs32_224"), ("c2_file_bs8", "gpt2_bs8_s128")):
        src = REPO / "tests" / "golden" / "traces"
        path = tdir / f"{name}.json"
        path.write_bytes(gzip.open(src / f"{name}.trace.json.gz").read())
        side = src / f"{name}.sidecar.json"
        est = eng.PeakMemoryEstimator()
        est.estimate(eng.parse_trace(path, sidecar=eng.load_sidecar(side)))  # warm
        times, rep = [], None
        for _ in range(5):
            t0 = time.perf_counter()
            rep = est.estimate(eng.parse_trace(path, sidecar=eng.load_sidecar(side)))
            times.append(time.perf_counter() - t0)
        out[key] = {"workload": f"{name}: trace file -> parse_trace -> "
                                "PeakMemoryEstimator.estimate -> report",
                    "file_mb": round(path.stat().st_size / 1e6, 1),
                    "ms": 1e3 * statistics.median(times),
                    "report_identical_to_reference": rep.canonical_json() ==
                    gold[name]["report_default"],
                    "timing": "wall clock, median of 5, warm"}
    # C5
    bundle = synth_events.generate(357200, 2)
    build_sequences([bundle], 2)  # warm (pool growth at this size)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    sb = build_sequences([bundle], 2)
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    b = DeviceBatch(sb.d_reqs, sb.req_off, cfg_record(AllocatorConfig()), device=dev.index)
    t2 = time.perf_counter()
    b.launch(stream)
    torch.cuda.synchronize(dev)
    t3 = time.perf_counter()
    res = b.results()
    out["c5"] = {"workload": "one C5-style event-level trace, 357200 leaf layers, "
                             "2 iterations", "events": len(bundle),
                 "requests": int(sb.req_off[-1]),
                 "analyze_build_sequence_s": t1 - t0,
                 "replay_s": t3 - t2, "status": int(res[0]["status"]),
                 "peak_reserved": int(res[0]["peak_reserved"]),
                 "timing": "wall clock around synchronised calls (batched pipeline "
                           "pm_pipeline_batch with B = 1; single-trace replay)"}
    return out


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
                           f"{dt1:.2f} s on 1 thread",
           **host_info()}
    parity = None
    if gpu_results is not None:
        mism = int((gpu_results[idx] != res).sum())
        parity = {"checked_traces": int(len(idx)), "mismatches": mism,
                  "fields": "all pm_result_t fields (peaks, finals, status, "
                            "stop index, segment counts, pool high-water)"}
    return out, parity


# ---- reference arm --------------------------------------------------------------

def run_reference(args, rank, world):
    """Reference arm: the reference algorithm's CPU implementation (the C
    port of allocator.py, oracle/replay_oracle.c) on the box's host cores,
    rank 0 only, on the engine arm's exact config.  Loads nothing but
    oracle/lib/liboracle_replay.so (which also holds the C3 generator)."""
    if rank != 0:
        return
    from oracle import replay as oracle
    threads = len(os.sched_getaffinity(0))
    ids = sweep_ids(args, world)
    stride = min(REF_STRIDE, len(ids))
    cfg = np.zeros(1, dtype=oracle.CFG_DTYPE)
    # AllocatorConfig() defaults (allocator.py:49-76); max_split / capacity None
    MIB = 1 << 20
    cfg[0] = (1 * MIB, 2 * MIB, 10 * MIB, 20 * MIB, 2 * MIB, 512, -1, -1)

    def sample(step):
        sel = ids[ids % stride == step % stride]
        return sel, oracle.c3_traces(sel, threads)

    times, events_total, covered = [], 0, set()
    for s in range(args.warmup + args.steps):
        sel, (reqs, offs) = sample(s)
        t0 = time.perf_counter()
        res, _ = oracle.replay_batch(reqs, offs, cfg, n_threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            events_total += int(res["n_events_replayed"].sum())
            covered.update((s % stride,))
    value = events_total / sum(times)
    sample_desc = (f"step s replays the {len(ids) // stride} traces i with "
                   f"i % {stride} == s % {stride}; the {args.steps} timed steps "
                   f"covered {len(covered)}/{stride} residues "
                   f"({events_total} requests in total)")
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded Llama-style request traces, SURVEY §8d C3)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads,
                         "kind": "port", "sample": sample_desc, **host_info()},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "implementation": "oracle/replay_oracle.c: C restatement of "
                          "peakmem.allocator (the reference is pure Python; "
                          "its own throughput is reported beside it)",
    }
    # the reference's own Python replay on 16 traces of the last sample,
    # each result checked against the port (pins the port live)
    k = min(16, len(offs) - 1)
    pick = np.linspace(0, len(offs) - 2, k).astype(np.int64)
    got = reference_replay(reqs, offs, pick, threads)
    if got is not None:
        ref_res, wall, ev, per_core = got
        line["reference_python"] = {
            "value": ev / wall, "unit": "events/s", "cores": min(threads, k),
            "per_core": per_core,
            "sample": f"{k} C3 traces ({ev} requests), peakmem.allocator "
                      "AllocatorState from baseline/_ref, one process per trace",
            "port_mismatches": int((res[pick] != ref_res).sum())}
    print(json.dumps(line))


# ---- dry run: the multi-rank host path on CPU -----------------------------------

def run_dry(args, rank, world):
    """gloo + oracle: shard (LPT), per-rank replay, gather in trace order,
    max-over-ranks time -- the engine arm's plumbing without a GPU."""
    import torch
    import torch.distributed as dist
    from oracle import replay as oracle
    from paper_2504_03887_b200.shard import gather_results, lpt_shards
    if world > 1:
        dist.init_process_group("gloo")
    else:
        dist = None
    ids = sweep_ids(args, world)
    all_reqs, all_offs = oracle.c3_traces(ids, 2)
    lengths = np.diff(all_offs)
    mine = (np.arange(rank * args.traces, (rank + 1) * args.traces)
            if args.weak else lpt_shards(lengths, world)[rank])
    reqs, offs = oracle.c3_traces(ids[mine], 2)
    cfg = np.zeros(1, dtype=oracle.CFG_DTYPE)
    MIB = 1 << 20
    cfg[0] = (1 * MIB, 2 * MIB, 10 * MIB, 20 * MIB, 2 * MIB, 512, -1, -1)
    t0 = time.perf_counter()
    res, _ = oracle.replay_batch(reqs, offs, cfg, n_threads=2)
    dt = time.perf_counter() - t0
    full = gather_results(res, mine, len(ids), dist)
    t = torch.tensor([dt], dtype=torch.float64)
    ev = torch.tensor([float(res["n_events_replayed"].sum())], dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
    ranks = _gather(dist, {"rank": rank, "traces": int(len(mine)),
                           "requests": int(offs[-1])}, world)
    if rank == 0:
        print(json.dumps({
            "dry_run": True, "metric": METRIC, "value": None, "unit": "events/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "scaling": "weak" if args.weak else "strong",
            "config": workload_config(args, world), "ranks": ranks,
            "requests_all_ranks": int(ev.item()), "max_rank_s": float(t.item()),
            "results_peak_reserved": full["peak_reserved"].tolist(),
            "results_n_events": full["n_events_replayed"].tolist()}))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
