"""Stage times of PeakMemoryEstimator.estimate_many on 64 C2-sized synthetic
bundles (GPU box): the whole call, then its parts alone -- the 64 config
digests (8 host threads), build_sequences, the replay batch.

    python tools/profile_many.py [traces] [leaves]
"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import logging
    logging.disable(logging.WARNING)
    import numpy as np
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as api
    from paper_2504_03887_b200 import synth_events
    from paper_2504_03887_b200.batch import build_sequences
    from paper_2504_03887_b200.engine import DeviceBatch
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    leaves = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
    bundles = [synth_events.generate(leaves + 7 * i, 2) for i in range(n)]
    ev = sum(len(b.start) for b in bundles)
    est = api.PeakMemoryEstimator()
    est.estimate_many(bundles[:2])

    def timed(f, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return round(best * 1e3, 2)

    out = {"traces": n, "events": ev}
    out["estimate_many_ms"] = timed(lambda: est.estimate_many(bundles))
    out["digests_8_threads_ms"] = timed(lambda: list(ThreadPoolExecutor(8).map(
        lambda b: est._digest(b, 0, 0), bundles)))
    out["digests_16_threads_ms"] = timed(lambda: list(ThreadPoolExecutor(16).map(
        lambda b: est._digest(b, 0, 0), bundles)))
    out["digest_one_ms"] = timed(lambda: est._digest(bundles[0], 0, 0))
    out["build_sequences_ms"] = timed(lambda: build_sequences(bundles, iterations=2))
    seqs = build_sequences(bundles, iterations=2)
    cfg = np.concatenate([cfg_record(AllocatorConfig())] * n)

    def replay():
        b = DeviceBatch(seqs.d_reqs, seqs.req_off, cfg, np.arange(n, dtype=np.int32),
                        device=seqs.d_reqs.device.index)
        b.launch()
        b.results()
    out["replay_batch_ms"] = timed(replay)
    out["requests"] = int(seqs.req_off[-1])
    print(out, flush=True)
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    est.estimate_many(bundles)
    pr.disable()
    pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
