"""C4 config sweep: GPT-2 capture sequences and C3 traces
under all 69 allocator configurations in one batch, every result field
against the C oracle (bit-exact)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from c4_cases import c4_batch, c4_configs
from conftest import GOLDEN
from oracle import replay as oracle

FIELDS = ("peak_reserved", "peak_allocated", "final_reserved",
          "final_allocated", "stop_index", "n_events_replayed", "status",
          "n_segments_final", "n_segments_peak", "max_free_blocks")


def test_grid_has_69_configs():
    cfgs = c4_configs()
    assert len(cfgs) == 69
    assert len({(c.max_split_size, c.alignment, c.k_small_buffer, c.k_large_buffer,
                 c.k_round_large) for c in cfgs}) == 69


def test_oracle_sweep_smoke():
    z = np.load(GOLDEN / "c2_sequences.npz")
    reqs, offs = z["reqs"], z["offsets"][:3]
    big, boffs, rec, cfg_of = c4_batch(reqs[:offs[-1]], offs, c4_configs())
    res, _ = oracle.replay_batch(big, boffs, rec, cfg_of)
    assert (res["status"] == 0).all()
    # configs change the answer (the sweep is not degenerate)
    assert len(set(res["peak_reserved"].tolist())) > 5


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_c4_sweep_gpu_matches_oracle():
    from paper_2504_03887_b200 import _native, synth
    z = np.load(GOLDEN / "c2_sequences.npz")
    r3, o3 = synth.generate(12, first=7000)
    reqs = np.concatenate([z["reqs"], r3])
    offs = np.concatenate([z["offsets"], o3[1:] + z["offsets"][-1]])
    big, boffs, rec, cfg_of = c4_batch(reqs, offs, c4_configs())
    want, _ = oracle.replay_batch(big, boffs, rec, cfg_of)
    got, _ = _native.replay_host(big, boffs, rec, cfg_of, False)
    for f in FIELDS:
        bad = np.nonzero(got[f] != want[f])[0]
        assert len(bad) == 0, (f, bad[:5].tolist())
