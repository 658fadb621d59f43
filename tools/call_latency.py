"""Per-call latency of the drop-in API on small sequences (GPU box):
paper_2504_03887_b200.replay vs the reference's peakmem.allocator.replay.

    python tools/call_latency.py
"""
import statistics
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def main():
    import torch  # noqa: F401
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    ref_root = REPO / "baseline" / "_ref"
    sys.path.insert(0, str(ref_root if (ref_root / "peakmem").exists()
                           else Path("/root/reference/pkg/src")))
    import peakmem.allocator as ref
    from replay_cases import corpus
    cases = corpus("corpus_seed1000")[:200]
    for impl, fn, cfgcls in (("engine", eng.replay, eng.AllocatorConfig),
                             ("reference", ref.replay, ref.AllocatorConfig)):
        times = []
        for seq, p in cases:
            cfg = cfgcls(device_capacity=p["capacity"], max_split_size=p["max_split_size"])
            t0 = time.perf_counter()
            fn(seq, cfg)
            times.append(time.perf_counter() - t0)
        n = sum(len(seq) for seq, _ in cases)
        print(f"{impl:9s} median {1e3 * statistics.median(times):.3f} ms/call, "
              f"total {sum(times):.3f} s for {len(cases)} calls ({n} requests)")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def profile():
    import cProfile
    import pstats
    import torch  # noqa: F401
    import paper_2504_03887_b200 as eng
    from replay_cases import corpus
    cases = corpus("corpus_seed1000")[:200]
    for seq, p in cases[:20]:
        eng.replay(seq, eng.AllocatorConfig(device_capacity=p["capacity"],
                                            max_split_size=p["max_split_size"]))
    pr = cProfile.Profile()
    pr.enable()
    for seq, p in cases:
        eng.replay(seq, eng.AllocatorConfig(device_capacity=p["capacity"],
                                            max_split_size=p["max_split_size"]))
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--profile":
    profile()
