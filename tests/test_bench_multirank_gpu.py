"""GPU: bench.py's multi-rank path with real replays on a one-GPU machine.

`--gpus 2` re-launches bench.py under torch.distributed.run; with
`--shared-device` both ranks replay their LPT shards of one sweep on cuda:0
and synchronise over gloo (the N-GPU path differs only in the device index
and the NCCL backend).  The line must report both ranks, every trace of the
sweep replayed once, and reference parity on rank 0's shard."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def test_two_ranks_on_one_gpu():
    cmd = [sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--shared-device",
           "--traces", "240", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
           "--no-other-configs", "--ref-check-traces", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["shared_device"]
    assert len(line["ranks"]) == 2
    assert sum(r["traces"] for r in line["ranks"]) == 240
    assert line["requests_per_step"] == sum(r["requests"] for r in line["ranks"])
    assert line["parity"]["reference_mismatches"] == 0
    assert line["value"] > 0 and line["e2e"]["value"] > 0
