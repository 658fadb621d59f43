"""Replay parity pinned to the REFERENCE beyond its default constants.

Goldens from tests/golden/make_golden_configs.py (the reference's own
AllocatorState, allocator.py:155-393): the C4 69-config grid
(replay_c4_grid.json), 400 multi-stream sequences with all eight allocator
knobs drawn and finite capacities in half (replay_multistream.json), and 32
full C3 traces at the bench config (replay_c3_full.json).  The C oracle is
checked on CPU; the engine on the GPU, every field plus timeline digests.
"""

from __future__ import annotations

import pytest

from config_goldens import c3_full_batch, c4_grid_batch, check, multistream_batch
from oracle import replay as oracle


def _oracle(batch):
    reqs, offs, cfgs, cfg_of, gold = batch
    res, tl = oracle.replay_batch(reqs, offs, cfgs, cfg_of, timeline=True)
    return check(res, tl, offs, gold)


def test_oracle_c4_grid():
    assert _oracle(c4_grid_batch()) == 690


def test_oracle_multistream():
    assert _oracle(multistream_batch()) == 400


def test_oracle_c3_full():
    assert _oracle(c3_full_batch(oracle.c3_traces)) == 32


def test_goldens_are_not_degenerate():
    from conftest import golden
    g = golden("replay_c4_grid.json")["results"]
    assert len({r["peak_reserved"] for r in g}) > 100
    m = golden("replay_multistream.json")["cases"]
    assert sum(c["oom_seq_no"] is not None for c in m) > 40
    assert sum(c["params"]["alignment"] != 512 for c in m) > 200


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestEngineAgainstReference:
    def _engine(self, batch):
        from paper_2504_03887_b200 import _native
        reqs, offs, cfgs, cfg_of, gold = batch
        res, tl = _native.replay_host(reqs, offs, cfgs, cfg_of, True)
        return check(res, tl, offs, gold)

    def test_c4_grid(self):
        assert self._engine(c4_grid_batch()) == 690

    def test_multistream(self):
        assert self._engine(multistream_batch()) == 400

    def test_c3_full(self):
        from paper_2504_03887_b200 import synth
        assert self._engine(c3_full_batch(synth.generate_ids)) == 32

    def test_c3_full_device_resident(self):
        """The bench's own path: DeviceBatch (pm_replay_batch on device
        buffers), no timeline."""
        import numpy as np
        from paper_2504_03887_b200 import synth
        from paper_2504_03887_b200.engine import DeviceBatch
        reqs, offs, cfg, _, gold = c3_full_batch(synth.generate_ids)
        b = DeviceBatch(reqs, offs, cfg, device=0)
        b.launch()
        check(b.results(), None, offs, gold)
        assert np.all(b.results()["status"] == 0)
