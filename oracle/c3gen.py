"""TEST INFRASTRUCTURE -- the C3 workload spec, restated with numpy.

SURVEY.md §8d, config C3: 10^4 request-level Llama-style training traces,
trace i drawn from ``numpy.random.Generator(PCG64(1_000_003 + i))``.  This
module is the executable specification of that recipe: it draws every random
number through numpy's own Generator (``integers`` / ``random``), in a fixed
order, and emits the requests in the order the reference's build_sequence
would orchestrate them (orchestration.py:237-399):

* model load at the head: the layer parameters, reversed (orchestration.py:
  135-161 -- permanent ALLOCs);
* per iteration: the previous iteration's gradients die at zero_grad
  (orchestration.py:187-197), a batch block (b*s*8 B) lives for the step
  (orchestration.py:164-184);
* forward, per layer: 10 retained activations (b*s*h*2 x6, b*s*ffn*2 x3,
  b*heads*s^2*2 x1) with an intra-op temporary after every third, plus one
  small temporary;
* backward, reverse layer order: a temporary around the weight gradients
  (the layer's parameter sizes, freed at the next zero_grad), a temporary
  between them, then the layer's activations freed in reverse;
* optimizer state, 2x the parameter sizes, allocated in iteration 0 only and
  never freed (orchestration.py:200-227);
* 10 % of activation / temporary sizes multiplied by U[0.5, 1.5], floored;
* iterations repeat until the trace holds at least its drawn target length
  (U{90000..110000} requests: 10^5 +- 10 %).

The product generator (workloads/c3gen.c, compiled into the engine's synth
library and, separately, into the oracle library for the reference bench
arm) reimplements PCG64 / SeedSequence / Generator.integers / random in C;
tests/test_c3gen.py pins it to this module trace for trace.
"""

from __future__ import annotations

import numpy as np

REQ_DTYPE = np.dtype([("size", "<i8"), ("handle", "<i4"),
                      ("kind_stream", "<u4")])
SEED_BASE = 1_000_003
NPARAM = 9
NACT = 10


def trace(index: int) -> np.ndarray:
    """Packed requests (size, handle, kind) of C3 trace `index`."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + index))
    L = (4, 8, 16, 32)[int(rng.integers(0, 4))]
    h = (1024, 2048, 3072, 4096)[int(rng.integers(0, 4))]
    ffn = 256 * -(-8 * h // 768)          # 256 * ceil(8h / 3 / 256)
    heads = h // 128
    b = int(rng.integers(1, 17))
    s = (256, 512, 1024, 2048)[int(rng.integers(0, 4))]
    target = int(rng.integers(90_000, 110_001))
    E = 2  # bf16
    psize = [h * h * E] * 4 + [h * ffn * E] * 3 + [h * E] * 2
    asize = [b * s * h * E] * 6 + [b * s * ffn * E] * 3 + [b * heads * s * s * E]

    sizes: list[int] = []
    handles: list[int] = []
    kinds: list[int] = []
    nh = [0]

    def alloc(size: int) -> int:
        hd = nh[0]
        nh[0] += 1
        sizes.append(size)
        handles.append(hd)
        kinds.append(0)
        return hd

    def free(hd: int) -> None:
        sizes.append(0)
        handles.append(hd)
        kinds.append(1)

    def jitter(size: int) -> int:
        if rng.random() < 0.1:
            return max(int(size * (0.5 + rng.random())), 1)
        return size

    for _ in range(L):                    # model load, reversed
        for p in reversed(range(NPARAM)):
            alloc(psize[p])
    acts = [0] * (L * NACT)
    grads = [0] * (L * NPARAM)
    have_grads = False
    it = 0
    while len(sizes) < target:
        if have_grads:                    # zero_grad
            for g in grads:
                free(g)
        batch = alloc(b * s * 8)
        for layer in range(L):            # forward
            for a in range(NACT):
                acts[layer * NACT + a] = alloc(jitter(asize[a]))
                if a % 3 == 2:
                    t = alloc(jitter(asize[0] if a < 6 else asize[6]))
                    free(t)
            k = int(rng.integers(0, 16))
            small = alloc(jitter(4096 + 512 * k))
            free(small)
        for layer in reversed(range(L)):  # backward
            t0 = alloc(jitter(asize[6]))
            for p in range(NPARAM):
                grads[layer * NPARAM + p] = alloc(psize[p])
                if p == 3:
                    t1 = alloc(jitter(asize[0]))
                    free(t1)
            free(t0)
            for a in reversed(range(NACT)):
                free(acts[layer * NACT + a])
            t2 = alloc(jitter(asize[0]))
            free(t2)
        have_grads = True
        if it == 0:                       # optimizer state, permanent
            for layer in range(L):
                for p in range(NPARAM):
                    alloc(psize[p])
                    alloc(psize[p])
        free(batch)
        it += 1
    out = np.empty(len(sizes), dtype=REQ_DTYPE)
    out["size"] = sizes
    out["handle"] = handles
    out["kind_stream"] = kinds
    return out
