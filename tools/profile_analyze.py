"""cProfile of analyze / build_sequence on a C5-scale event trace (GPU box).

    python tools/profile_analyze.py [leaves]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch  # noqa: F401
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    leaves = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
    b0 = synth_events.generate(2000, 2)
    api.build_sequence(api.analyze(b0), 2)  # warm-up (CUDA context, libraries)
    b = synth_events.generate(leaves, 2)
    for _ in range(2):
        t0 = time.perf_counter()
        a = api.analyze(b)
        t1 = time.perf_counter()
        api.build_sequence(a, 2)
        t2 = time.perf_counter()
        print(f"analyze {t1 - t0:.3f} s  build_sequence {t2 - t1:.3f} s", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    a = api.analyze(b)
    api.build_sequence(a, 2)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
