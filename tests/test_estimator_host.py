"""CPU: the estimator's host-side orchestration (no GPU needed) -- the
config digest runs on a host thread beside the device pipeline, and errors
surface in the reference's order (estimator.py:135-179): analysis / replay
errors first, a digest error only where the reference computes the digest.
"""

from __future__ import annotations

import pytest

from paper_2504_03887_b200 import estimator as est_mod
from paper_2504_03887_b200.estimator import PeakMemoryEstimator, _Background


def test_background_returns_value_and_reraises():
    assert _Background(lambda a, b: a + b, 2, 3).result() == 5
    with pytest.raises(KeyError, match="boom"):
        _Background(lambda: {}["boom"]).result()


def test_analysis_error_wins_over_digest_error(monkeypatch):
    class Analysis(Exception):
        pass

    def bad_analyze(bundle):
        raise Analysis("analysis")

    monkeypatch.setattr(est_mod, "analyze", bad_analyze)
    monkeypatch.setattr(PeakMemoryEstimator, "_digest",
                        lambda self, *a: (_ for _ in ()).throw(ValueError("digest")))

    class Bundle:
        metadata = None

    with pytest.raises(Analysis):
        PeakMemoryEstimator().estimate_with_details(Bundle(), _timeline=False)


def test_digest_error_surfaces_after_the_pipeline(monkeypatch):
    calls = []

    class Seq:
        def breakdown(self):
            return {}

        def __len__(self):
            return 0

    class Res:
        peak_reserved = peak_allocated = 0
        oom_seq_no = None

    monkeypatch.setattr(est_mod, "analyze", lambda b: calls.append("analyze"))
    monkeypatch.setattr(est_mod, "build_sequence",
                        lambda a, iterations: calls.append("build") or Seq())
    monkeypatch.setattr(est_mod, "replay_sequence",
                        lambda s, cfg, timeline=True, validate=False: calls.append(("replay", timeline)) or Res())
    monkeypatch.setattr(PeakMemoryEstimator, "_digest",
                        lambda self, *a: (_ for _ in ()).throw(ValueError("digest")))

    class Bundle:
        metadata = None

    with pytest.raises(ValueError, match="digest"):
        PeakMemoryEstimator().estimate_with_details(Bundle(), _timeline=False)
    # the whole device pipeline ran first; no timeline was asked for
    assert calls == ["analyze", "build", ("replay", False)]


class _FakeSeqs:
    """batch.SequenceBatch stand-in: per-trace errors, empty sequences."""

    def __init__(self, errors):
        import numpy as np
        self.errors = errors
        self.req_off = np.zeros(len(errors) + 1, np.int64)

        class _Dev:  # stands in for a device tensor: only .device.index is read
            class device:
                index = 0
        self.d_reqs = _Dev()

    def breakdown(self, t):
        return {}

    def packed(self, t):
        return None


def _fake_device_batch(calls):
    import numpy as np
    from paper_2504_03887_b200._native import RESULT_DTYPE

    class DB:
        def __init__(self, reqs, offs, cfgs, cfg_of, device=0):
            self.n = len(offs) - 1

        def launch(self):
            calls.append("replay")

        def results(self):
            return np.zeros(self.n, RESULT_DTYPE)

    return DB


def test_estimate_many_pipeline_error_wins_over_digest_error(monkeypatch):
    from paper_2504_03887_b200 import batch, engine

    class Analysis(Exception):
        pass

    calls = []
    monkeypatch.setattr(batch, "build_sequences",
                        lambda b, iterations: _FakeSeqs([None, Analysis("a")]))
    monkeypatch.setattr(engine, "DeviceBatch", _fake_device_batch(calls))
    monkeypatch.setattr(PeakMemoryEstimator, "_digest",
                        lambda self, *a: (_ for _ in ()).throw(ValueError("digest")))

    class Bundle:
        metadata = None

    # trace 0 succeeds up to its digest, which raises first (bundle order)
    with pytest.raises(ValueError, match="digest"):
        PeakMemoryEstimator().estimate_many([Bundle(), Bundle()])
    got = PeakMemoryEstimator().estimate_many([Bundle(), Bundle()],
                                              return_exceptions=True)
    assert isinstance(got[0], ValueError) and isinstance(got[1], Analysis)
    # a failing pipeline alone: its error, never the digest's
    monkeypatch.setattr(batch, "build_sequences",
                        lambda b, iterations: _FakeSeqs([Analysis("a")]))
    with pytest.raises(Analysis):
        PeakMemoryEstimator().estimate_many([Bundle()])


def test_estimate_many_digest_error_after_replay(monkeypatch):
    from paper_2504_03887_b200 import batch, engine
    calls = []
    monkeypatch.setattr(batch, "build_sequences",
                        lambda b, iterations: calls.append("build") or _FakeSeqs([None]))
    monkeypatch.setattr(engine, "DeviceBatch", _fake_device_batch(calls))
    monkeypatch.setattr(PeakMemoryEstimator, "_digest",
                        lambda self, *a: (_ for _ in ()).throw(ValueError("digest")))

    class Bundle:
        metadata = None

    with pytest.raises(ValueError, match="digest"):
        PeakMemoryEstimator().estimate(Bundle())
    assert calls == ["build", "replay"]


def test_estimate_many_of_no_bundles_is_empty():
    # parameters are still validated; nothing reaches the device
    assert PeakMemoryEstimator().estimate_many([]) == []
    with pytest.raises(ValueError):
        PeakMemoryEstimator(iterations=0).estimate_many([])
