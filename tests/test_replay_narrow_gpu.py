"""GPU parity at the edges of the narrow encoding (csrc/replay_narrow.cuh).

The main pass holds sizes and addresses in allocator units u = 2^s as
32-bit values; a trace that leaves that range (another stream, a block or
an address space of >= 2^32 - 1 units, a unit above 16 MiB) stops and is
replayed from the start by the wide tiers.  Every case here is checked
against the C oracle (oracle/replay_oracle.c, the restatement of
allocator.py:155-393 pinned to the reference's corpora) with full
timelines, so the hand-off itself is what is tested.
"""

from __future__ import annotations

import os
import random
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import replay as oracle
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]

MIB = 1 << 20
GIB = 1 << 30
REPO = Path(__file__).resolve().parent.parent


def alloc(seq, bid, size, **kw):
    return {"seq_no": seq, "kind": "alloc", "block_id": bid, "size": size, **kw}


def free(seq, bid):
    return {"seq_no": seq, "kind": "free", "block_id": bid}


def run_both(traces, cfgs):
    packed = [pack_trace(t) for t in traces]
    offs = np.zeros(len(traces) + 1, dtype=np.int64)
    np.cumsum([len(p.reqs) for p in packed], out=offs[1:])
    reqs = np.concatenate([p.reqs for p in packed])
    carr = np.concatenate([cfg_record(c) for c in cfgs])
    cof = np.arange(len(traces), dtype=np.int32)
    got, tl = _native.replay_host(reqs, offs, carr, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, carr, cof, timeline=True)
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} traces differ, first {bad[:5]}: " \
        f"{got[bad[0]]} vs {want[bad[0]]}"
    assert (tl == tl_ref).all()
    # the same batch through the 8-byte wire format, where it encodes
    words = _native.wire_pack(reqs, offs)
    if words is not None:
        gw, tlw = _native.replay_host_wire(words, offs, carr, cof, True)
        assert (gw == want).all() and (tlw == tl_ref).all()
    return got


def test_address_space_past_2tib_escalates():
    # 12 GiB segments never freed: next_base passes 2^32 units of 512 B
    # (2 TiB) part-way through, the narrow pass hands the trace over
    seq, k = [], 0
    for i in range(200):
        seq.append(alloc(k, i, 12 * GIB + 513)); k += 1
        if i % 3 == 0:
            seq.append(alloc(k, 1000 + i, 4096)); k += 1
    small = [alloc(0, 0, 4096), free(1, 0)]
    got = run_both([seq, small], [AllocatorConfig(), AllocatorConfig()])
    assert got[0]["peak_reserved"] > (1 << 41)


def test_block_at_unit_limit():
    # one request just below / at / above the largest narrow block
    u = 512
    lim = (0xFFFFFFFE * u)
    traces = [[alloc(0, 0, lim - u), alloc(1, 1, 600), free(2, 0), alloc(3, 2, 1000)],
              [alloc(0, 0, lim), free(1, 0)],
              [alloc(0, 0, lim + 1), free(1, 0), alloc(2, 1, 512)],
              [alloc(0, 0, 1 << 45), free(1, 0)]]
    run_both(traces, [AllocatorConfig(k_round_large=512)] * len(traces))


def test_odd_segment_sizes_unit_one():
    # k_small_buffer odd -> u = 1 B: 4 GiB of segments already leaves the
    # encoding; small traces stay narrow
    rng = random.Random(17)
    cfg = AllocatorConfig(k_small_buffer=2 * MIB + 1, alignment=1)
    traces = []
    for n in (40, 300, 2000):
        live, seq, nxt = [], [], 0
        for _ in range(n):
            if live and rng.random() < 0.4:
                seq.append(free(len(seq), live.pop(rng.randrange(len(live)))))
            else:
                seq.append(alloc(len(seq), nxt, rng.choice(
                    [rng.randint(1, 3 * MIB), rng.randint(1, 900 * MIB)])))
                live.append(nxt)
                nxt += 1
        traces.append(seq)
    run_both(traces, [cfg] * len(traces))


def test_huge_unit_goes_wide():
    # unit 2^26 B (> 2^24): the whole trace runs in the wide tiers
    cfg = AllocatorConfig(alignment=1 << 26, k_small_buffer=1 << 27,
                          k_large_buffer=1 << 28, k_round_large=1 << 27,
                          k_small_size=1 << 27, k_min_large_alloc=1 << 28)
    seq = [alloc(0, 0, 5), alloc(1, 1, 1 << 27), free(2, 0), alloc(3, 2, 7),
           free(3, 1), free(4, 2)]
    run_both([seq], [cfg])


def test_error_before_escalation_wins():
    # a duplicate handle before the first out-of-range request is reported
    # by the narrow pass; the reverse order by the wide tiers
    a = [alloc(0, 0, 512), alloc(1, 0, 512), alloc(2, 1, 1 << 44)]
    b = [alloc(0, 0, 512), alloc(1, 1, 1 << 44), alloc(2, 0, 512)]
    c = [alloc(0, 0, 512), alloc(1, 1, 512, stream=2), free(2, 5)]
    got = run_both([a, b, c], [AllocatorConfig()] * 3)
    assert list(got["status"]) == [4, 4, 2]


def test_mixed_batch_split_thresholds_and_capacity():
    # C3 traces with split thresholds that are not unit multiples and a
    # capacity that forces releases, next to escalating multistream traces
    reqs, offs = synth.generate(12, first=3000)
    cfgs = np.concatenate([
        cfg_record(AllocatorConfig(max_split_size=20 * MIB + 77)),
        cfg_record(AllocatorConfig(max_split_size=64 * MIB, alignment=4096)),
        cfg_record(AllocatorConfig(device_capacity=24 * GIB + 5)),
        cfg_record(AllocatorConfig(max_split_size=32 * MIB + 1,
                                   device_capacity=20 * GIB))])
    cof = (np.arange(12) % 4).astype(np.int32)
    got, tl = _native.replay_host(reqs, offs, cfgs, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfgs, cof, timeline=True)
    assert (got == want).all()
    assert (tl == tl_ref).all()


def _wire_ok(seq):
    p = pack_trace(seq)
    return _native.wire_pack(p.reqs, np.array([0, len(p.reqs)])) is not None


def test_wire_format_corpus_and_synthetic_vs_oracle():
    # every corpus trace the wire format encodes, plus C3 traces with split
    # thresholds and capacities (OOM verdicts), through pm_replay_host_wire
    from replay_cases import corpus, pack_corpus
    cases = corpus("corpus_seed1000")
    r, o, c, f, _ = pack_corpus(cases)
    keep = [i for i in range(len(o) - 1)
            if _native.wire_pack(r[o[i]:o[i + 1]], np.array([0, o[i + 1] - o[i]]))
            is not None]
    assert len(keep) > 200
    parts = [r[o[i]:o[i + 1]] for i in keep]
    offs = np.zeros(len(keep) + 1, dtype=np.int64)
    np.cumsum([len(x) for x in parts], out=offs[1:])
    reqs = np.concatenate(parts)
    cof = f[keep]
    words = _native.wire_pack(reqs, offs)
    got, tl = _native.replay_host_wire(words, offs, c, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, c, cof, timeline=True)
    assert (got == want).all() and (tl == tl_ref).all()
    assert (want["status"] == 1).sum() > 50  # OOM verdicts among them

    reqs, offs = synth.generate(16, first=4000)
    cfgs = np.concatenate([cfg_record(AllocatorConfig()),
                           cfg_record(AllocatorConfig(max_split_size=64 * MIB)),
                           cfg_record(AllocatorConfig(device_capacity=20 * GIB))])
    cof = (np.arange(16) % 3).astype(np.int32)
    words = _native.wire_pack(reqs, offs)
    assert words is not None
    got, tl = _native.replay_host_wire(words, offs, cfgs, cof, True)
    want, tl_ref = oracle.replay_batch(reqs, offs, cfgs, cof, timeline=True)
    assert (got == want).all() and (tl == tl_ref).all()


def test_wire_format_escalations_expand_for_wide_tiers():
    # wire traces that leave the narrow pass (> 32 buckets of free blocks;
    # > 2 TiB of segments) are expanded to pm_req_t for the wide tiers
    holes = [alloc(i, i, 512) for i in range(3000)]
    holes += [free(3000 + k, 2 * k) for k in range(1500)]
    holes += [alloc(4500 + k, 3000 + k, 512) for k in range(700)]
    big, k = [], 0
    for i in range(200):
        big.append(alloc(k, i, 12 * GIB + 513)); k += 1
    assert _wire_ok(holes) and _wire_ok(big)
    run_both([holes, big, [alloc(0, 0, 4096), free(1, 0)]],
             [AllocatorConfig()] * 3)


_WIDE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import replay as oracle
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
from replay_cases import corpus, pack_corpus
r, o, c, f, _ = pack_corpus(corpus("corpus_seed1000")[:400])
got, tl = _native.replay_host(r, o, c, f, True)
want, tl_ref = oracle.replay_batch(r, o, c, f, timeline=True)
assert (got == want).all() and (tl == tl_ref).all()
reqs, offs = synth.generate(16, first=77)
cfg = cfg_record(AllocatorConfig())
got, _ = _native.replay_host(reqs, offs, cfg, None, False)
want, _ = oracle.replay_batch(reqs, offs, cfg)
assert (got == want).all()
print("wide ok")
"""


@pytest.mark.parametrize("env", [{"PM_REPLAY_WIDE": "1"},
                                 {"PM_REPLAY_WARPS": "12"},
                                 {"PM_REPLAY_WARPS": "20"},
                                 {"PM_REPLAY_WARPS": "32"}])
def test_main_kernel_variants_vs_oracle(env):
    # the wide main kernel (PM_REPLAY_WIDE=1) and the other narrow widths;
    # the launch configuration is fixed per process, hence a subprocess
    code = _WIDE_SCRIPT.format(repo=str(REPO), tests=str(REPO / "tests"))
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "wide ok" in out.stdout


def _permuted_trace(rng, n_allocs):
    """Raw pm_req_t records whose dense handles are NOT in first-appearance
    order (the C ABI allows any dense handles), with a few malformed
    requests: frees of never-allocated handles, double frees, duplicates."""
    perm = rng.permutation(2 * n_allocs)  # handles < n_requests
    recs, live, used = [], [], []
    _permuted_trace.unused = int(perm[n_allocs])  # a handle never allocated
    for k in range(n_allocs):
        h = int(perm[k])
        recs.append((int(rng.integers(1, 64 << 20)), h, 0))
        live.append(h)
        used.append(h)
        while live and rng.random() < 0.45:
            recs.append((0, live.pop(int(rng.integers(len(live)))), 1))
    for h in live:
        recs.append((0, h, 1))
    out = np.array(recs, dtype=_native.REQ_DTYPE)
    return out


def test_out_of_order_handles_and_dirty_workspace_vs_oracle():
    # the handle watermark must zero the records it jumps over; a second
    # launch over the same (dirty) workspace must not trust old records
    rng = np.random.default_rng(99)
    traces = [_permuted_trace(rng, m) for m in (3, 40, 700, 5000)]
    bad = []
    for kind in range(3):  # unknown handle, double free, duplicate alloc
        t = _permuted_trace(rng, 300).copy()
        i = len(t) // 2
        if kind == 0:
            h = _permuted_trace.unused
            t = np.concatenate([t[:i], np.array([(0, h, 1)], t.dtype), t[i:]])
        elif kind == 1:
            f = np.nonzero(t["kind_stream"][:i] == 1)[0][-1]
            t = np.concatenate([t[:i], t[f:f + 1], t[i:]])
        else:
            a = np.nonzero(t["kind_stream"][:i] == 0)[0][-1]
            t = np.concatenate([t[:i], t[a:a + 1], t[i:]])
        bad.append(t)
    traces += bad
    offs = np.zeros(len(traces) + 1, dtype=np.int64)
    np.cumsum([len(t) for t in traces], out=offs[1:])
    reqs = np.concatenate(traces)
    assert (reqs["handle"] < np.repeat(np.diff(offs), np.diff(offs))).all()
    cfg = cfg_record(AllocatorConfig())
    want, tl_ref = oracle.replay_batch(reqs, offs, cfg, timeline=True)
    assert set(want["status"][-3:].tolist()) == {2, 3, 4}
    from paper_2504_03887_b200.engine import DeviceBatch
    batch = DeviceBatch(reqs, offs, cfg, timeline=True)
    for _ in range(2):
        batch.launch()
        assert (batch.results() == want).all()
        tlb = batch.timeline().ravel()
        assert (tlb[:tl_ref.size] == tl_ref.ravel()).all()
    got, tl = _native.replay_host(reqs, offs, cfg, None, True)
    assert (got == want).all() and (tl == tl_ref).all()


@pytest.mark.parametrize("host_copy", ["0", "1"])
def test_pinned_host_buffers_zero_copy_and_streamed(host_copy, monkeypatch):
    # pinned requests are read in place by the kernel (zero copy) or, with
    # PM_HOST_COPY=1, streamed by the copy engines behind the launched main
    # pass; both entry points, full timelines, vs the oracle
    import torch
    monkeypatch.setenv("PM_HOST_COPY", host_copy)
    reqs, offs = synth.generate(40, first=7000)
    cfgs = np.concatenate([cfg_record(AllocatorConfig()),
                           cfg_record(AllocatorConfig(max_split_size=64 * MIB,
                                                      device_capacity=24 * GIB))])
    cof = (np.arange(40) % 2).astype(np.int32)
    pin = torch.empty(len(reqs) * 16, dtype=torch.uint8, pin_memory=True)
    preqs = pin.numpy().view(_native.REQ_DTYPE)
    preqs[:] = reqs
    wpin = torch.empty(len(reqs) * 8, dtype=torch.uint8, pin_memory=True)
    words = _native.wire_pack(preqs, offs, out=wpin.numpy().view(np.uint64))
    want, tl_ref = oracle.replay_batch(reqs, offs, cfgs, cof, timeline=True)
    got, tl = _native.replay_host(preqs, offs, cfgs, cof, True)
    assert (got == want).all() and (tl == tl_ref).all()
    got, tl = _native.replay_host_wire(words, offs, cfgs, cof, True)
    assert (got == want).all() and (tl == tl_ref).all()


_STARVED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import replay as oracle
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
from paper_2504_03887_b200.engine import DeviceBatch
reqs, offs = synth.generate(300, first=2000)
cfg = cfg_record(AllocatorConfig())
want, _ = oracle.replay_batch(reqs, offs, cfg)
b = DeviceBatch(reqs, offs, cfg)
b.launch()
assert (b.results() == want).all()
print("starved ok", b.tier_counts())
"""


def test_starved_shared_pool_waits_and_escalates_vs_oracle():
    # a 48-bucket pool for 24 warps: warps wait for buckets, deadlocked CTAs
    # give up one victim at a time; every result must still be the oracle's
    code = _STARVED_SCRIPT.format(repo=str(REPO), tests=str(REPO / "tests"))
    out = subprocess.run([sys.executable, "-c", code],
                         env={**os.environ, "PM_POOL_BUCKETS": "48"},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "starved ok" in out.stdout
