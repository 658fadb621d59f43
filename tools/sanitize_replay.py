"""Small replay batches for compute-sanitizer (racecheck / memcheck):
C3 traces through the main pass, corpus traces with capacities and split
thresholds, hole traces through the retry passes, wire words zero-copy;
batches of at most one trace per SM run the one-warp main-pass CTA, the
300-trace batch the 12-warp one (PM_SPREAD=0: every batch in 24-warp CTAs).

    compute-sanitizer --tool racecheck python tools/sanitize_replay.py
"""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def main():
    import torch  # noqa: F401
    from oracle import replay as oracle
    from paper_2504_03887_b200 import _native, synth
    from paper_2504_03887_b200.allocator import AllocatorConfig, cfg_record, pack_trace
    from replay_cases import corpus, pack_corpus
    reqs, offs = synth.generate(6, first=123)
    cfg = cfg_record(AllocatorConfig())
    got, _ = _native.replay_host(reqs, offs, cfg, None, True)
    want, _ = oracle.replay_batch(reqs, offs, cfg)
    assert (got == want).all()
    r, o, c, f, _ = pack_corpus(corpus("corpus_seed1000")[:120])
    got, _ = _native.replay_host(r, o, c, f, True)
    want, _ = oracle.replay_batch(r, o, c, f)
    assert (got == want).all()
    holes = [{"seq_no": i, "kind": "alloc", "block_id": i, "size": 512} for i in range(3000)]
    holes += [{"seq_no": 3000 + k, "kind": "free", "block_id": 2 * k} for k in range(1500)]
    p = pack_trace(holes)
    o2 = np.array([0, len(p.reqs)], np.int64)
    got, _ = _native.replay_host(p.reqs, o2, cfg, None, True)
    want, _ = oracle.replay_batch(p.reqs, o2, cfg)
    assert (got == want).all()
    words = _native.wire_pack(reqs, offs)
    got, _ = _native.replay_host_wire(words, offs, cfg, None, False)
    want, _ = oracle.replay_batch(reqs, offs, cfg)
    assert (got == want).all()
    # a batch of more than one trace per SM: the 12-warp main-pass CTA
    r, o, c, f, _ = pack_corpus(corpus("corpus_seed1000")[:300])
    got, _ = _native.replay_host(r, o, c, f, True)
    want, _ = oracle.replay_batch(r, o, c, f)
    assert (got == want).all()
    print("sanitize batches ok")


if __name__ == "__main__":
    main()
