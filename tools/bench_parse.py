"""Trace-reader throughput on C2-sized input without capturing: K copies of
the committed GPT-2 bs8 capture (21.6 MB each) parsed with parse_trace,
serially and from host thread pools (as tools/bench_c2_e2e.py does).

    python tools/bench_parse.py [copies]
"""
import gzip
import os
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor
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
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    g = REPO / "tests" / "golden" / "traces"
    data = gzip.open(g / "gpt2_bs8_s128.trace.json.gz").read()
    side = eng.load_sidecar(g / "gpt2_bs8_s128.sidecar.json")
    d = Path(tempfile.mkdtemp())
    files = []
    for i in range(k):
        f = d / f"t{i}.json"
        f.write_bytes(data)
        files.append(f)
    mb = len(data) * k / 1e6

    def parse(f):
        return eng.parse_trace(f, sidecar=side)

    parse(files[0])
    out = {"files": k, "mb": round(mb, 1), "cores": os.cpu_count()}
    t0 = time.perf_counter()
    for f in files[:8]:
        parse(f)
    out["serial_ms_per_file"] = round((time.perf_counter() - t0) / 8 * 1e3, 2)
    for w in (8, 16):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            with ThreadPoolExecutor(max_workers=w) as pool:
                list(pool.map(parse, files))
            best = min(best, time.perf_counter() - t0)
        out[f"pool{w}_s"] = round(best, 3)
        out[f"pool{w}_gbs"] = round(mb / 1e3 / best, 2)
    print(out, flush=True)


if __name__ == "__main__":
    main()
