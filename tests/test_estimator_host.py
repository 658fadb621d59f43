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
        PeakMemoryEstimator().estimate(Bundle())


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
        PeakMemoryEstimator().estimate(Bundle())
    # the whole device pipeline ran first; estimate() asks for no timeline
    assert calls == ["analyze", "build", ("replay", False)]
