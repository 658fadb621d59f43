"""traces x the 69-config allocator grid (max_split_size x
alignment x segment-size set, minus the combinations AllocatorConfig rejects,
allocator.py:73-76), replayed as one batch with one config per replica."""

from __future__ import annotations

import numpy as np

MIB = 1 << 20


def c4_configs():
    from paper_2504_03887_b200.allocator import AllocatorConfig
    seg_sets = [{}, {"k_small_buffer": 4 * MIB}, {"k_large_buffer": 32 * MIB},
                {"k_round_large": 4 * MIB}]
    out = []
    for ms in (None, 20 * MIB, 32 * MIB, 64 * MIB, 128 * MIB, 256 * MIB):
        for al in (512, 1024, 4096):
            for seg in seg_sets:
                try:
                    out.append(AllocatorConfig(max_split_size=ms, alignment=al, **seg))
                except ValueError:  # max_split below the large buffer
                    continue
    return out


def c4_batch(reqs, offs, cfgs):
    """Every trace replicated once per config: (reqs, offsets, cfg records,
    cfg_of) -- replica r = trace r // len(cfgs), config r % len(cfgs)."""
    from paper_2504_03887_b200.allocator import cfg_record
    n, m = len(offs) - 1, len(cfgs)
    lens = np.diff(offs)
    parts = []
    for t in range(n):
        seg = reqs[offs[t]:offs[t + 1]]
        parts.extend([seg] * m)
    big = np.concatenate(parts)
    boffs = np.zeros(n * m + 1, np.int64)
    np.cumsum(np.repeat(lens, m), out=boffs[1:])
    rec = np.concatenate([cfg_record(c) for c in cfgs])
    cfg_of = np.tile(np.arange(m, dtype=np.int32), n)
    return big, boffs, rec, cfg_of
