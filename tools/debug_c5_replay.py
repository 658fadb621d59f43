"""Which replay tier does the single C5 trace take, and how fast?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
import paper_2504_03887_b200 as api
from paper_2504_03887_b200 import synth_events
from paper_2504_03887_b200.allocator import cfg_record
from paper_2504_03887_b200.engine import DeviceBatch
leaves = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
b = synth_events.generate(leaves, 2)
seq = api.build_sequence(api.analyze(b), 2)
reqs = seq.packed
offs = np.array([0, len(reqs)], np.int64)
batch = DeviceBatch(reqs, offs, cfg_record(api.AllocatorConfig()))
for _ in range(2):
    t = time.perf_counter(); batch.launch(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    r = batch.results()
    ctl = batch.d_ws[:64].cpu().numpy().view(np.uint32)
    print(f"{len(reqs)} requests {dt:.2f} s  {len(reqs)/dt/1e6:.2f} Mreq/s passes {ctl[9:15]} maxF {r['max_free_blocks'][0]} nseg {r['n_segments_peak'][0]} status {r['status'][0]}")
