"""TEST INFRASTRUCTURE -- synthetic CPU-profiler traces (chrome-trace records).

Generates traces shaped like the reference's captures (pkg/capture/capture.py:
a model trained under torch.profiler with profile_memory / with_stack /
with_modules): nested `nn.Module: ` python_function frames with python ids
and parent links, cpu_op intervals carrying sequence numbers (forward ops
inside module frames, backward `autograd::engine::evaluate_function` ops
outside them, nested child ops), `[memory]` instants whose addresses are
recycled through a size-keyed free list (so alloc/free pairing by address
recurrence is exercised), and ProfilerStep / zero_grad / Optimizer.step
annotations.  Deterministic per seed; used to build golden vectors with the
reference (tests/golden/make_golden_pipeline.py) and as parity inputs on the
GPU box.
"""

from __future__ import annotations

import random


def generate(seed: int, iterations: int = 3, layers: int = 6, leaves: int = 3,
             optimizer: str = "adam", zero_grad: str = "start",
             jitter_ts: bool = True) -> tuple[list[dict], dict]:
    """Return (chrome records, sidecar dict)."""
    rng = random.Random(seed)
    recs: list[dict] = []
    t = 1_000_000.0 + rng.random() * 1000
    pyid = [1000]
    seq = [0]
    free_addrs: dict[int, list[int]] = {}
    next_addr = [0x7f0000000000]

    def tick(lo=1.0, hi=5.0):
        nonlocal t
        t += rng.uniform(lo, hi) if jitter_ts else lo
        return t

    def new_addr(size):
        lst = free_addrs.get(size)
        if lst and rng.random() < 0.8:
            return lst.pop(rng.randrange(len(lst)))
        a = next_addr[0]
        next_addr[0] += ((size + 511) // 512) * 512 + 512 * rng.randint(0, 3)
        return a

    def instant(ts, addr, nbytes):
        recs.append({"ph": "i", "cat": "cpu_instant_event", "name": "[memory]",
                     "ts": round(ts, 3), "s": "t",
                     "args": {"Addr": addr, "Bytes": nbytes,
                              "Total Allocated": 0, "Total Reserved": 0}})

    def alloc(size, ts=None):
        a = new_addr(size)
        instant(ts if ts is not None else tick(0.1, 0.5), a, size)
        return (a, size)

    def free(blk, ts=None):
        a, size = blk
        instant(ts if ts is not None else tick(0.1, 0.5), a, -size)
        free_addrs.setdefault(size, []).append(a)

    def frame(cat, name, ts, dur, args=None):
        rec = {"ph": "X", "cat": cat, "name": name, "ts": round(ts, 3),
               "dur": round(dur, 3), "args": args or {}}
        recs.append(rec)
        return rec

    def pyfunc(name, ts, dur, parent=None):
        pyid[0] += 1
        args = {"Python id": pyid[0]}
        if parent is not None:
            args["Python parent id"] = parent
        frame("python_function", name, ts, dur, args)
        return pyid[0]

    hidden = rng.choice([64, 128, 256])
    param_sizes = []
    for _ in range(layers):
        for _ in range(leaves):
            param_sizes += [hidden * hidden * 4, hidden * 4]
    batch = rng.choice([2, 4, 8])
    batch_bytes = [batch * hidden * 4, batch * 8]
    grads_live: list = []
    state_allocated = False

    # a non-layer python frame that owns the whole run (root of the chain)
    for it in range(iterations):
        step_start = tick(5, 10)
        step_rec = frame("user_annotation", f"ProfilerStep#{it}", step_start, 0)
        if zero_grad == "start":
            zs = tick()
            for g in grads_live:
                free(g, tick(0.1, 0.3))
            frame("user_annotation", "Optimizer.zero_grad#Adam.zero_grad",
                  zs, t - zs + 1)
            grads_live = []
        # forward: Model > Block_l > Leaf_j frames
        acts = []
        model_start = tick()
        top = pyfunc("train.py(42): train_step", model_start - 0.5, 0)
        mid = pyfunc("nn.Module: Model_0", model_start, 0, parent=top)
        fwd_seqs = []
        for l in range(layers):
            bs = tick()
            blk = pyfunc(f"nn.Module: Block_{l}", bs, 0, parent=mid)
            for j in range(leaves):
                ls = tick()
                helper = pyfunc("torch/nn/modules/module.py(1500): _call_impl",
                                ls, 0, parent=blk)
                leaf = pyfunc(f"nn.Module: Linear_{l}_{j}", tick(0.2, 0.5), 0,
                              parent=helper)
                del leaf
                op_s = tick(0.2, 0.6)
                seq[0] += 1
                fwd_seqs.append(seq[0])
                act = alloc(batch * hidden * 4 * rng.choice([1, 1, 2]))
                acts.append(act)
                tmp = alloc(batch * hidden * 4)
                child_s = tick(0.1, 0.3)
                frame("cpu_op", "aten::addmm", child_s, rng.uniform(0.5, 1.5),
                      {"Sequence number": seq[0] if rng.random() < 0.3 else -1})
                tick(1.5, 2.0)
                free(tmp)
                op_e = tick(0.2, 0.6)
                frame("cpu_op", "aten::linear", op_s, op_e - op_s,
                      {"Sequence number": seq[0]})
                if rng.random() < 0.2:  # an unowned small block
                    alloc(512)
                le = tick(0.2, 0.5)
                # patch leaf / helper frame durations
                for r in reversed(recs):
                    if r.get("cat") == "python_function" and \
                            r["args"].get("Python id") in (helper, helper + 1):
                        r["dur"] = round(le - r["ts"], 3)
                tick(0.2, 0.4)
            be = tick()
            for r in reversed(recs):
                if r.get("cat") == "python_function" and r["args"].get("Python id") == blk:
                    r["dur"] = round(be - r["ts"], 3)
                    break
        me = tick()
        for r in reversed(recs):
            if r.get("cat") == "python_function" and r["args"].get("Python id") in (mid, top):
                r["dur"] = round(me - r["ts"] + (0.5 if r["args"]["Python id"] == top else 0), 3)
        if zero_grad == "pre-backward":
            zs = tick()
            for g in grads_live:
                free(g, tick(0.1, 0.3))
            frame("user_annotation", "Optimizer.zero_grad#Adam.zero_grad",
                  zs, t - zs + 1)
            grads_live = []
        # backward: evaluate_function ops carry the forward sequence numbers
        loss = alloc(4)
        for k, s in enumerate(reversed(fwd_seqs)):
            op_s = tick()
            g1 = alloc(hidden * hidden * 4)
            g2 = alloc(hidden * 4)
            grads_live += [g1, g2]
            if rng.random() < 0.5:
                tmp = alloc(batch * hidden * 4)
                tick()
                free(tmp)
            free(acts[len(acts) - 1 - k])
            op_e = tick()
            frame("cpu_op", "autograd::engine::evaluate_function: AddmmBackward0",
                  op_s, op_e - op_s, {"Sequence number": s})
            if rng.random() < 0.3:  # nested op inside the backward op
                frame("cpu_op", "aten::mm", op_s + 0.01, (op_e - op_s) / 2,
                      {"Sequence number": -1})
        free(loss)
        # optimizer step
        os_ = tick()
        if optimizer == "adam" and not state_allocated:
            for ps in param_sizes:
                alloc(ps)
                alloc(ps)
            state_allocated = True
        for _ in range(3):
            tmp = alloc(rng.choice(param_sizes))
            free(tmp)
        oe = tick()
        frame("user_annotation", "Optimizer.step#Adam.step", os_, oe - os_)
        step_rec["dur"] = round(tick() - step_start, 3)
    recs.append({"ph": "M", "name": "process_name", "args": {"name": "x"}})
    rng.shuffle(recs)  # file order is not time order
    sidecar = {"param_sizes": param_sizes, "batch_bytes": batch_bytes,
               "optimizer": optimizer, "device_capacity_bytes": 0,
               "initial_memory_bytes": 0}
    return recs, sidecar
