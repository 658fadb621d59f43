"""CPU, world size 2 over gloo: the multi-GPU host path of a sweep --
LPT shards are disjoint, cover every trace and balance the load; every rank
replays its own shard (the C oracle stands in for the device on CPU) and the
per-trace results gather back in trace order EQUAL to a one-process replay
of the whole sweep; the step time reduces as a max over ranks (bench.py's
rule); and `bench.py --gpus 2 --dry-run` spawns its own two ranks."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03887_b200.shard import gather_results, lpt_shards

from conftest import REPO
from oracle import replay as oracle

MIB = 1 << 20


def _cfg():
    cfg = np.zeros(1, dtype=oracle.CFG_DTYPE)
    cfg[0] = (1 * MIB, 2 * MIB, 10 * MIB, 20 * MIB, 2 * MIB, 512, -1, -1)
    return cfg


SWEEP = np.arange(500, 524, dtype=np.int32)   # 24 C3 traces


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    reqs_all, offs_all = oracle.c3_traces(SWEEP, 2)
    lengths = np.diff(offs_all)
    mine = lpt_shards(lengths, world)[rank]
    # replay the shard (oracle on CPU; pm_replay_batch on a GPU rank)
    reqs, offs = oracle.c3_traces(SWEEP[mine], 2)
    local, _ = oracle.replay_batch(reqs, offs, _cfg(), n_threads=2)
    full = gather_results(local, mine, len(lengths), dist)
    t = torch.tensor([float(100 + rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    load = torch.tensor([int(lengths[mine].sum())], dtype=torch.int64)
    loads = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(loads, load)
    if rank == 0:
        q.put((full.tobytes(), float(t.item()), [int(x.item()) for x in loads],
               lengths.tolist()))
    dist.destroy_process_group()


def test_lpt_shards_single_process():
    lengths = np.array([5, 9, 1, 7, 7, 3])
    parts = lpt_shards(lengths, 3)
    assert sorted(np.concatenate(parts).tolist()) == list(range(6))
    loads = sorted(int(lengths[p].sum()) for p in parts)
    assert loads[-1] - loads[0] <= lengths.max()


def test_two_rank_gloo_sweep():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    full_b, tmax, loads, lengths = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.frombuffer(full_b, dtype=oracle.RESULT_DTYPE)
    lengths = np.array(lengths)
    reqs, offs = oracle.c3_traces(SWEEP, 2)
    single, _ = oracle.replay_batch(reqs, offs, _cfg(), n_threads=2)
    assert (full == single).all()
    assert (full["n_events_replayed"] == lengths).all()
    assert tmax == 101.0
    assert sum(loads) == lengths.sum()
    assert abs(loads[0] - loads[1]) <= lengths.max()


def test_bench_spawns_two_ranks_dry_run():
    """bench.py --gpus 2 without torchrun launches 2 ranks itself; the
    gathered per-trace results equal a one-process replay of the sweep."""
    env = dict(os.environ, PYTHONPATH=str(REPO))
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(
        [sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--dry-run",
         "--traces", "24", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, env=env, cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines()
                       if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert [r["rank"] for r in line["ranks"]] == [0, 1]
    assert sum(r["traces"] for r in line["ranks"]) == 24
    reqs, offs = oracle.c3_traces(np.arange(24, dtype=np.int32), 2)
    single, _ = oracle.replay_batch(reqs, offs, _cfg(), n_threads=2)
    assert line["results_peak_reserved"] == single["peak_reserved"].tolist()
    assert line["requests_all_ranks"] == int(offs[-1])
