"""cProfile of the per-trace API (analyze + build_sequence) at C5 size."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    leaves = int(sys.argv[1]) if len(sys.argv) > 1 else 357200
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    b = synth_events.generate(leaves, 2)
    api.build_sequence(api.analyze(b), 2)
    torch.cuda.synchronize()
    for _ in range(2):
        t0 = time.perf_counter()
        a = api.analyze(b)
        t1 = time.perf_counter()
        api.build_sequence(a, 2)
        torch.cuda.synchronize()
        print(f"analyze {t1 - t0:.4f} s  build_sequence {time.perf_counter() - t1:.4f} s", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    api.build_sequence(api.analyze(b), 2)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
