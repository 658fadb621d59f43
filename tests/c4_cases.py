"""traces x the 69-config allocator grid (max_split_size x
alignment x segment-size set, minus the combinations AllocatorConfig rejects,
allocator.py:73-76), replayed as one batch with one config per replica."""

from __future__ import annotations

import numpy as np

MIB = 1 << 20


def c4_grid_params():
    """AllocatorConfig kwargs of the 69 grid points."""
    seg_sets = [{}, {"k_small_buffer": 4 * MIB}, {"k_large_buffer": 32 * MIB},
                {"k_round_large": 4 * MIB}]
    out = []
    for ms in (None, 20 * MIB, 32 * MIB, 64 * MIB, 128 * MIB, 256 * MIB):
        for al in (512, 1024, 4096):
            for seg in seg_sets:
                # AllocatorConfig rejects max_split below the large buffer
                # (allocator.py:73-76)
                if ms is not None and ms < seg.get("k_large_buffer", 20 * MIB):
                    continue
                out.append({"max_split_size": ms, "alignment": al, **seg})
    return out


def c4_configs(config_cls=None):
    if config_cls is None:
        from paper_2504_03887_b200.allocator import AllocatorConfig as config_cls
    return [config_cls(**p) for p in c4_grid_params()]


def timeline_digest(tl_pairs, seq_nos=None) -> str:
    """sha256 over int64 rows (seq_no, reserved, allocated) -- the compact
    timeline digest of the configuration goldens."""
    import hashlib
    tl_pairs = np.asarray(tl_pairs, dtype=np.int64).reshape(-1, 2)
    if seq_nos is None:
        seq_nos = np.arange(len(tl_pairs), dtype=np.int64)
    rows = np.column_stack([np.asarray(seq_nos, dtype=np.int64), tl_pairs])
    return hashlib.sha256(rows.astype("<i8").tobytes()).hexdigest()


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
