"""GPU: the C ABI from a plain C host (tests/c_abi/replay_smoke.c, built
with gcc against include/peakmem_b200.h and the in-tree library) -- the
drop-in boundary without Python -- against the oracle."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import replay as oracle
from paper_2504_03887_b200 import _native
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record

REPO = Path(__file__).resolve().parent.parent
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]
MIB = 1 << 20


def test_c_host_matches_oracle(tmp_path):
    lib = _native.LIB_PATH
    exe = tmp_path / "replay_smoke"
    subprocess.run(["gcc", "-O2", "-I", str(REPO / "include"),
                    str(REPO / "tests" / "c_abi" / "replay_smoke.c"), "-o", str(exe),
                    "-L", str(lib.parent), "-lpeakmem_b200", f"-Wl,-rpath,{lib.parent}"],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True,
                         env={**os.environ, "LD_LIBRARY_PATH": str(lib.parent)})
    got = [list(map(int, ln.split())) for ln in out.stdout.strip().splitlines()]
    # the same requests through the oracle
    A = lambda s, h: (s, h, 0)  # noqa: E731
    F = lambda h: (0, h, 1)  # noqa: E731
    recs = [A(1 * MIB, 0), A(3 * MIB, 1), A(700 * 1024, 2), F(0), A(512 * 1024, 3),
            F(2), F(3), A(25 * MIB, 4), F(1), A(2 * MIB, 5), F(4), F(5),
            A(10 * MIB, 0), A(10 * MIB, 1), F(0), A(30 * MIB, 2), A(40 * MIB, 3)]
    reqs = np.zeros(len(recs), _native.REQ_DTYPE)
    reqs["size"] = [r[0] for r in recs]
    reqs["handle"] = [r[1] for r in recs]
    reqs["kind_stream"] = [r[2] for r in recs]
    offs = np.array([0, 12, 17], np.int64)
    cfgs = np.concatenate([cfg_record(AllocatorConfig()),
                           cfg_record(AllocatorConfig(device_capacity=64 * MIB))])
    want, _ = oracle.replay_batch(reqs, offs, cfgs, np.array([0, 1], np.int32))
    exp = [[int(w["status"]), int(w["peak_reserved"]), int(w["peak_allocated"]),
            int(w["final_reserved"]), int(w["final_allocated"]),
            int(w["n_segments_peak"]), int(w["stop_index"])] for w in want]
    assert got == exp
    assert got[1][0] == 1  # the capacity trace ends in an OOM verdict
