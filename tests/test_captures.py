"""Real training-step captures (SURVEY §8d C1 ResNet-18 bs32, C2 GPT-2 small
batch sweep): pipeline views + reports (GPU) and replay of the orchestrated
GPT-2 sequences at 2 and 10 iterations (GPU batch and CPU oracle), all
against the reference's outputs (tests/golden/make_golden_captures.py)."""

from __future__ import annotations

import gzip
import json
import logging

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import replay as oracle
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record

logging.disable(logging.WARNING)
FIELDS = ("peak_reserved", "peak_allocated", "final_reserved",
          "final_allocated", "n_segments_final", "n_segments_peak",
          "max_free_blocks")


def c2():
    z = np.load(GOLDEN / "c2_sequences.npz")
    return z["reqs"], z["offsets"], json.loads(str(z["meta"]))


def check_results(res, meta):
    for r, m in zip(res, meta):
        assert int(r["status"]) == 0, m["name"]
        for f in FIELDS:
            assert int(r[f]) == m[f], (m["name"], m["iterations"], f)


def test_c2_sequences_oracle():
    reqs, offs, meta = c2()
    res, _ = oracle.replay_batch(reqs, offs, cfg_record(AllocatorConfig()))
    check_results(res, meta)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_c2_sequences_gpu_batch():
    from paper_2504_03887_b200 import _native
    reqs, offs, meta = c2()
    res, _ = _native.replay_host(reqs, offs, cfg_record(AllocatorConfig()), None, False)
    check_results(res, meta)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
@pytest.mark.parametrize("name", ["resnet18_bs32_224", "gpt2_bs8_s128"])
def test_capture_pipeline_matches_reference(name, tmp_path):
    import paper_2504_03887_b200 as api
    from pipeline_cases import views
    trace = tmp_path / f"{name}.json"
    with gzip.open(GOLDEN / "traces" / f"{name}.trace.json.gz", "rb") as f:
        trace.write_bytes(f.read())
    side = api.load_sidecar(GOLDEN / "traces" / f"{name}.sidecar.json")
    got = views(api, api.parse_trace(trace, sidecar=side))
    want = golden("captures_golden.json")[name]
    for key in want:
        assert got[key] == want[key], key


# ---- C2 as BASELINE.json states it: 64 GPT-2 small traces, bs 1..64 --------

def c2_sweep():
    z = np.load(GOLDEN / "c2_sweep.npz")
    return z["reqs"], z["offsets"], golden("c2_sweep_golden.json")["traces"]


def check_sweep(res, tl, offs, meta):
    from conftest import digest
    assert len(meta) == 64 and [m["batch"] for m in meta] == list(range(1, 65))
    check_results(res, meta)
    for i, m in enumerate(meta):
        assert int(res[i]["n_events_replayed"]) == m["n_requests"] == m["timeline_len"]
        if tl is not None:
            pairs = tl[2 * offs[i]: 2 * offs[i + 1]].reshape(-1, 2).tolist()
            rows = [[k, a, b] for k, (a, b) in enumerate(pairs)]
            assert digest(rows) == m["timeline_sha256"], m["name"]


def test_c2_sweep_oracle():
    reqs, offs, meta = c2_sweep()
    res, tl = oracle.replay_batch(reqs, offs, cfg_record(AllocatorConfig()),
                                  timeline=True)
    check_sweep(res, tl, offs, meta)
    # the sweep is what it claims: 64 different peaks growing with batch size
    peaks = [m["peak_reserved"] for m in meta]
    assert len(set(peaks)) == 64 and peaks[-1] > 8 * peaks[0]


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_c2_sweep_gpu_one_batch():
    """All 64 orchestrated GPT-2 sequences replayed as ONE batch on the GPU,
    bit-exact against the reference (peaks, finals, segment counts, full
    timelines)."""
    from paper_2504_03887_b200 import _native
    reqs, offs, meta = c2_sweep()
    res, tl = _native.replay_host(reqs, offs, cfg_record(AllocatorConfig()), None, True)
    check_sweep(res, tl, offs, meta)
