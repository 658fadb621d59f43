"""One warm PeakMemoryEstimator.estimate on a committed capture (GPU box),
for launch lists: `ncu --metrics gpu__time_duration.sum --csv ... python
tools/one_estimate.py resnet18_bs32_224`.

    python tools/one_estimate.py [capture]
"""
import gzip
import logging
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    logging.disable(logging.WARNING)
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2504_03887_b200 as eng
    g = REPO / "tests" / "golden" / "traces"
    name = sys.argv[1] if len(sys.argv) > 1 else "resnet18_bs32_224"
    path = Path(tempfile.mkdtemp()) / "t.json"
    path.write_bytes(gzip.open(g / f"{name}.trace.json.gz").read())
    b = eng.parse_trace(path, sidecar=eng.load_sidecar(g / f"{name}.sidecar.json"))
    est = eng.PeakMemoryEstimator()
    for _ in range(3):
        est.estimate(b)
    torch.cuda.synchronize()
    t = time.perf_counter()
    est.estimate(b)
    torch.cuda.synchronize()
    print(f"{name}: estimate {(time.perf_counter() - t) * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
