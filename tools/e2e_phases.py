"""Time pm_replay_host phases on the C3 workload (PM_TRACE_PHASES=1)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["PM_TRACE_PHASES"] = "1"


def main():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03887_b200 import _native, synth
    from paper_2504_03887_b200._native import REQ_DTYPE
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    _, offs = synth.generate(1)  # warm
    counts_only = synth.generate(n, out=None)
    reqs, offs = counts_only
    pinned = torch.empty(len(reqs) * 16, dtype=torch.uint8, pin_memory=True)
    buf = pinned.numpy().view(REQ_DTYPE)
    buf[:] = reqs
    cfg = cfg_record(AllocatorConfig())
    wpin = torch.empty(len(reqs) * 8, dtype=torch.uint8, pin_memory=True)
    words = _native.wire_pack(buf, offs, out=wpin.numpy().view(np.uint64))
    for mode in ("1", "0"):  # PM_HOST_COPY: copy engines / zero copy
      os.environ["PM_HOST_COPY"] = mode
      for name, fn, src in (("pm_replay_host", _native.replay_host, buf),
                            ("pm_replay_host_wire", _native.replay_host_wire, words)):
        for _ in range(3):
            t0 = time.perf_counter()
            res, _ = fn(src, offs, cfg, None, False)
            dt = time.perf_counter() - t0
            print(f"PM_HOST_COPY={mode} {name}: wall {dt*1e3:.1f} ms  "
                  f"{len(reqs)/dt/1e9:.3f} Gev/s", flush=True)


if __name__ == "__main__":
    main()
