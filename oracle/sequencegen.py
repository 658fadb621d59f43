"""TEST INFRASTRUCTURE -- restated random request-sequence corpus.

The reference's parity corpus generator (pkg/src/peakmem/sequencegen.py:
random_sequence 15-40, random_config 43-51) restated so the corpus can be
regenerated where the reference tree is absent (the GPU box).  It must draw
from `random.Random` in exactly the reference's order; tests/golden pins
that with a digest of every generated sequence
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import random

MIB = 1 << 20

# sizes where the allocator's branches flip (sequencegen.py:33-35)
_BOUNDARY_SIZES = (1, 511, 512, 513, MIB, MIB + 1, 2 * MIB, 10 * MIB,
                   10 * MIB + 1, 20 * MIB)


def random_sequence(rng: random.Random, max_requests: int = 200,
                    max_size: int = 64 * MIB) -> list[dict]:
    """Well-formed alloc/free list: frees name live handles only, no reuse.

    Draw order per request (sequencegen.py:21-39): free-or-alloc coin
    (short-circuited when nothing is live or > 40 are live), then either a
    victim index or a size plus the 30 % boundary-size override.
    """
    count = rng.randint(1, max_requests)
    live: list[int] = []
    out: list[dict] = []
    fresh = 0
    while len(out) < count:
        if live and (rng.random() < 0.45 or len(live) > 40):
            k = rng.randrange(len(live))
            live[k], live[-1] = live[-1], live[k]
            out.append({"seq_no": len(out), "kind": "free",
                        "block_id": live.pop()})
            continue
        size = rng.randint(1, max_size)
        if rng.random() < 0.3:
            size = rng.choice(_BOUNDARY_SIZES)
        out.append({"seq_no": len(out), "kind": "alloc",
                    "block_id": fresh, "size": size})
        live.append(fresh)
        fresh += 1
    return out


def random_config(rng: random.Random) -> dict:
    """capacity: None or U[20 MiB, 512 MiB] (p=.5); max_split_size: None or
    U[20 MiB, 128 MiB] (p=.4) -- sequencegen.py:43-51."""
    capacity = rng.randint(20 * MIB, 512 * MIB) if rng.random() < 0.5 else None
    max_split = rng.randint(20 * MIB, 128 * MIB) if rng.random() < 0.4 else None
    return {"capacity": capacity, "max_split_size": max_split}


def corpus(seed: int, count: int) -> list[tuple[list[dict], dict]]:
    """(sequence, params) pairs, drawn like the reference's equivalence
    tests: sequence first, then config (test_acceptance.py:107-110)."""
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        seq = random_sequence(rng)
        out.append((seq, random_config(rng)))
    return out


def corpus_config_first(seed: int, count: int) -> list[tuple[list[dict], dict]]:
    """Config drawn before the sequence (test_allocator.py:201-205)."""
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        params = random_config(rng)
        out.append((random_sequence(rng), params))
    return out
