"""GPU: pm_replay_host on a large pinned pm_req_t batch packs the records to
8-byte wire words on host threads while the kernels replay them
(csrc/replay.cu replay_host_packed).  Results must equal the plain
zero-copy path (PM_HOST_PACK=0) and the oracle, including traces the wire
format cannot hold (a second stream, a duplicate handle, an unknown kind),
which are replayed again from their records."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import replay as oracle
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def _pinned_copy(reqs):
    import torch
    t = torch.empty(reqs.nbytes, dtype=torch.uint8, pin_memory=True)
    out = t.numpy().view(_native.REQ_DTYPE)
    out[:] = reqs
    return t, out


def _run(reqs, offs, cfgs, cfg_of, monkeypatch, pack):
    monkeypatch.setenv("PM_HOST_PACK", "1" if pack else "0")
    res, _ = _native.replay_host(reqs, offs, cfgs, cfg_of, False)
    return res


def test_packed_equals_zero_copy_and_oracle(monkeypatch):
    reqs, offs = synth.generate(40, first=321)
    assert offs[-1] >= 1 << 20  # large enough for the packed path
    keep, pinned = _pinned_copy(reqs)
    cfgs = np.concatenate([cfg_record(AllocatorConfig()),
                           cfg_record(AllocatorConfig(device_capacity=6 << 30,
                                                      max_split_size=64 << 20))])
    cfg_of = (np.arange(len(offs) - 1) % 2).astype(np.int32)
    got = _run(pinned, offs, cfgs, cfg_of, monkeypatch, True)
    plain = _run(pinned, offs, cfgs, cfg_of, monkeypatch, False)
    want, _ = oracle.replay_batch(reqs, offs, cfgs, cfg_of)
    assert (got == plain).all()
    assert (got == want).all()


def test_packed_falls_back_for_unencodable_traces(monkeypatch):
    reqs, offs = synth.generate(24, first=777)
    reqs = reqs.copy()
    # trace 3: a request on stream 1; trace 7: a duplicate handle; trace 11:
    # an unknown kind -- none has a wire encoding
    a3 = int(offs[3]) + 5
    reqs["kind_stream"][a3] = (reqs["kind_stream"][a3] & 3) | (1 << 2)
    a7 = int(offs[7])
    allocs7 = np.nonzero((reqs["kind_stream"][a7:offs[8]] & 3) == 0)[0]
    reqs["handle"][a7 + allocs7[3]] = reqs["handle"][a7 + allocs7[2]]
    reqs["kind_stream"][int(offs[11]) + 9] = 2
    keep, pinned = _pinned_copy(reqs)
    cfgs = cfg_record(AllocatorConfig())
    got = _run(pinned, offs, cfgs, None, monkeypatch, True)
    want, _ = oracle.replay_batch(reqs, offs, cfgs)
    assert (got == want).all()
    assert int(got["status"][7]) != 0 and int(got["status"][11]) != 0
