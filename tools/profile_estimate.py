"""cProfile of PeakMemoryEstimator.estimate on a C5-style bundle (GPU box).

    python tools/profile_estimate.py [leaves]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import logging
    logging.disable(logging.WARNING)
    import torch  # noqa: F401
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    leaves = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
    api.PeakMemoryEstimator(iterations=2).estimate(synth_events.generate(2000, 2))
    b = synth_events.generate(leaves, 2)
    t0 = time.perf_counter()
    api.PeakMemoryEstimator(iterations=2).estimate(b)
    print(f"estimate {time.perf_counter() - t0:.3f} s", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    api.PeakMemoryEstimator(iterations=2).estimate(b)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
