"""CPU, world size 2 over gloo: the multi-GPU host path of a sweep --
LPT shards are disjoint, cover every trace and balance the load; per-trace
results gather back in trace order; the step time reduces as a max over
ranks (bench.py's rule)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03887_b200.shard import gather_results, lpt_shards

DT = np.dtype([("peak", "<i8"), ("trace", "<i8")])


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
    rng = np.random.default_rng(3)
    lengths = rng.integers(90_000, 110_000, size=101)
    mine = lpt_shards(lengths, world)[rank]
    # "replay" the shard: a deterministic per-trace result
    local = np.zeros(len(mine), dtype=DT)
    local["peak"] = lengths[mine] * 7
    local["trace"] = mine
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
    full_b, tmax, loads, lengths = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.frombuffer(full_b, dtype=DT)
    lengths = np.array(lengths)
    assert (full["trace"] == np.arange(len(lengths))).all()
    assert (full["peak"] == lengths * 7).all()
    assert tmax == 101.0
    assert sum(loads) == lengths.sum()
    assert abs(loads[0] - loads[1]) <= lengths.max()
