"""cProfile of the batched pipeline (build_sequences) on one C5-style trace.

    python tools/profile_batch.py [leaves]
"""
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
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.batch import build_sequences
    b = synth_events.generate(leaves, 2)
    print(f"{len(b)} events", flush=True)
    build_sequences([b], 2)
    torch.cuda.synchronize()
    for _ in range(2):
        t0 = time.perf_counter()
        sb = build_sequences([b], 2)
        torch.cuda.synchronize()
        print(f"build_sequences {time.perf_counter() - t0:.4f} s, "
              f"{int(sb.req_off[-1])} requests", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    build_sequences([b], 2)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
