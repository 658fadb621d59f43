"""Find traces whose result depends on being a warp's 2nd trace."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_2504_03887_b200 import synth, _native
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
from oracle import replay as oracle

cfg = cfg_record(AllocatorConfig())
reqs, offs = synth.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
want, _ = oracle.replay_batch(reqs, offs, cfg)
got, _ = _native.replay_host(reqs, offs, cfg, None, False)
bad = np.nonzero(got != want)[0]
print("grid", os.environ.get("PM_MAX_GRID"), "mismatching traces:", bad.tolist()[:20])
for t in bad[:3]:
    print(" trace", t, "len", offs[t+1]-offs[t])
    print("  got ", got[t])
    print("  want", want[t])
