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


# --- corpus beyond the reference's own generator ----------------------------
# The reference's random_sequence draws stream 0 and default allocator
# constants only.  These corpora exercise the other knobs of AllocatorConfig
# (allocator.py:49-76: segment sizing :86-92, alignment) and the per-stream
# pool (allocator.py:163-165,176-178); tests/golden/make_golden_configs.py
# replays them through the REFERENCE and commits the results.

_SMALL_SIZE = (1 * MIB, 256 * 1024, 3 * MIB, MIB + 512)
_SMALL_BUF = (2 * MIB, 4 * MIB, 3 * MIB, 3 * MIB + 8192)
_MIN_LARGE = (10 * MIB, 8 * MIB, 16 * MIB, 5 * MIB)
_LARGE_BUF = (20 * MIB, 32 * MIB, 16 * MIB, 24 * MIB + 8192)
_ROUND_LARGE = (2 * MIB, 4 * MIB, 1 * MIB, 3 * MIB)
_ALIGN = (512, 1024, 4096, 256, 16, 8192)


def random_allocator_config(rng: random.Random) -> dict:
    """All eight AllocatorConfig knobs, kept in the regime a caching
    allocator is configured in: segments at least as large as the requests
    they serve, segment sizes multiples of the alignment (otherwise the
    reference itself fails its `remainder >= alignment` assertion in _split,
    allocator.py:225); AllocatorConfig's own validation always passes."""
    small = rng.choice(_SMALL_SIZE)
    small_buf = max(rng.choice(_SMALL_BUF), small)
    min_large = max(rng.choice(_MIN_LARGE), small)
    large_buf = max(rng.choice(_LARGE_BUF), min_large)
    cfg = {"k_small_size": small, "k_small_buffer": small_buf,
           "k_min_large_alloc": min_large, "k_large_buffer": large_buf,
           "k_round_large": rng.choice(_ROUND_LARGE),
           "alignment": rng.choice(_ALIGN)}
    cfg["max_split_size"] = (rng.randint(large_buf, 256 * MIB)
                             if rng.random() < 0.5 else None)
    cfg["device_capacity"] = (rng.randint(8 * MIB, 512 * MIB)
                              if rng.random() < 0.5 else None)
    return cfg


def multistream_sequence(rng: random.Random, cfg: dict,
                         max_requests: int = 300, streams: int = 4) -> list[dict]:
    """Well-formed sequence over `streams` streams; sizes straddle the
    config's own branch points 40 % of the time."""
    edges = [1, cfg["alignment"] - 1, cfg["alignment"], cfg["alignment"] + 1,
             cfg["k_small_size"], cfg["k_small_size"] + 1,
             cfg["k_min_large_alloc"], cfg["k_min_large_alloc"] + 1,
             cfg["k_large_buffer"], cfg["k_round_large"] + 1]
    if cfg["max_split_size"] is not None:
        edges += [cfg["max_split_size"] - 1, cfg["max_split_size"] + 1]
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
        size = rng.randint(1, 48 * MIB) if rng.random() < 0.6 else rng.randint(1, 2 * MIB)
        if rng.random() < 0.4:
            size = max(1, rng.choice(edges))
        stream = 0 if rng.random() < 0.5 else rng.randrange(streams)
        out.append({"seq_no": len(out), "kind": "alloc", "block_id": fresh,
                    "size": size, "stream": stream})
        live.append(fresh)
        fresh += 1
    return out


def multistream_corpus(seed: int, count: int) -> list[tuple[list[dict], dict]]:
    """(sequence, full AllocatorConfig kwargs) pairs: config drawn first."""
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        cfg = random_allocator_config(rng)
        out.append((multistream_sequence(rng, cfg), cfg))
    return out
