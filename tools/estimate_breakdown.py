"""Stage times of one captured trace through the engine (GPU box):
parse_trace, analyze, build_sequence, replay, digest.

    python tools/estimate_breakdown.py [capture]
"""
import gzip
import statistics
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    import logging
    logging.disable(logging.WARNING)
    import torch  # noqa: F401
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    from paper_2504_03887_b200.allocator import AllocatorConfig
    from paper_2504_03887_b200.estimator import replay_sequence
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2_bs8_s128"
    g = REPO / "tests" / "golden" / "traces"
    path = Path(tempfile.mkdtemp()) / "t.json"
    path.write_bytes(gzip.open(g / f"{name}.trace.json.gz").read())
    side = eng.load_sidecar(g / f"{name}.sidecar.json")
    est = eng.PeakMemoryEstimator()
    rows = []
    for _ in range(7):
        t = [time.perf_counter()]
        b = eng.parse_trace(path, sidecar=side)
        t.append(time.perf_counter())
        a = eng.analyze(b)
        t.append(time.perf_counter())
        s = eng.build_sequence(a, 2)
        t.append(time.perf_counter())
        replay_sequence(s, AllocatorConfig(), timeline=False)
        t.append(time.perf_counter())
        est._digest(b, 0, 0)
        t.append(time.perf_counter())
        rows.append([t[i + 1] - t[i] for i in range(5)])
    med = [statistics.median(r[i] for r in rows[2:]) for i in range(5)]
    print(name, {k: round(1e3 * v, 2) for k, v in zip(
        ("parse_ms", "analyze_ms", "build_sequence_ms", "replay_ms", "digest_ms"), med)},
        "requests", len(s))


if __name__ == "__main__":
    main()
