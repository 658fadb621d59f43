"""Run the 2-trace reproducer against the uniformity-checking debug build."""
import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2504_03887_b200 import _native, synth
from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record
from oracle import replay as oracle
lib = _native.load_library(_native.LIB_DIR / "libpeakmem_b200_debug.so")
_native._lib = lib
lib.pm_debug_nonuniform_line.restype = ctypes.c_int
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reqs, offs = synth.generate(n)
cfg = cfg_record(AllocatorConfig())
got, _ = _native.replay_host(reqs, offs, cfg, None, False)
want, _ = oracle.replay_batch(reqs, offs, cfg)
print("mismatch", np.nonzero(got != want)[0].tolist(), "first non-uniform line", lib.pm_debug_nonuniform_line())
