"""Pool-operation counters of the narrow kernel (debug build, -DPM_STATS).

    python tools/stats_replay.py [n_traces]
"""
import ctypes
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
NAMES = ["rekey in place", "rekey moved", "remove", "remove fill-hole", "bucket erase",
         "insert", "split", "merge", "best-fit scan", "best-fit next bucket",
         "argmin multi-candidate", "argmin key tie", "bucket alloc (bitmap)",
         "bucket wait round", "alloc miss (segment)", "free, no free neighbour"]


def main():
    import torch
    out = "/tmp/libpeakmem_stats.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-DPM_STATS", f"-I{REPO/'include'}", "-shared",
                    str(REPO / "paper_2504_03887_b200/csrc/replay.cu"), "-o", out], check=True)
    from paper_2504_03887_b200 import _native, synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    lib = _native.load_library(out)
    _native._lib = lib
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    if n < 0:  # C5: one event-level trace of -n leaves, orchestrated
        import paper_2504_03887_b200 as api
        from paper_2504_03887_b200 import synth_events
        seq = api.build_sequence(api.analyze(synth_events.generate(-n, 2)), 2)
        reqs = seq.packed
        offs = np.array([0, len(reqs)], dtype=np.int64)
    else:
        reqs, offs = synth.generate(n)
    res, _ = _native.replay_host(reqs, offs, cfg_record(AllocatorConfig()), None, False)
    st = (ctypes.c_ulonglong * 16)()
    lib.pm_debug_stats(st)
    ev = int(res["n_events_replayed"].sum())
    print(f"{n} traces, {ev} requests")
    for i, name in enumerate(NAMES):
        print(f"{name:24s} {st[i] / ev:8.4f} per request")


if __name__ == "__main__":
    main()
