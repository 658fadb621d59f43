"""Event-level synthetic traces at scale, built directly as a columnar
TraceBundle (one very long trace stressing the
interval joins and pool fragmentation).

Layout per iteration: `leaves` leaf modules, each a python_function layer
frame ("nn.Module: Linear_k") under a helper frame under a model frame; a
forward root op per leaf with a sequence number and two nested child ops;
the leaf's activation alloc (freed in backward) and an intra-op temporary;
backward root ops (same sequence numbers, outside the frames) allocating two
gradients each and freeing the activation; an optimizer-step span with
first-iteration state; ProfilerStep / zero_grad annotations.  Addresses are
recycled per size so alloc/free pairing by address recurrence is exercised.
Vectorised with numpy; ~16 events per leaf per iteration.
"""

from __future__ import annotations

import numpy as np

from .trace import (CATEGORY_CODES, EventCategory, NONE, NameColumn,
                    SidecarConfig, TraceBundle)

PF = CATEGORY_CODES[EventCategory.PYTHON_FUNCTION]
OP = CATEGORY_CODES[EventCategory.CPU_OP]
UA = CATEGORY_CODES[EventCategory.USER_ANNOTATION]
IN = CATEGORY_CODES[EventCategory.CPU_INSTANT_EVENT]

NAMES = ["nn.Module: Model_0", "module.py(1): _call_impl", "aten::linear",
         "aten::addmm", "aten::t",
         "autograd::engine::evaluate_function: AddmmBackward0", "aten::mm",
         "Optimizer.step#AdamW.step", "Optimizer.zero_grad#AdamW.zero_grad",
         "[memory]"]


def generate(leaves: int, iterations: int = 2, seed: int = 7,
             hidden: int = 256) -> TraceBundle:
    rng = np.random.default_rng(seed)
    cols = {k: [] for k in ("cat", "start", "dur", "name", "pid", "parent",
                            "seq", "addr", "nbytes")}
    names = list(NAMES)
    leaf_name0 = len(names)
    names += [f"nn.Module: Linear_{k}" for k in range(leaves)]
    step_name0 = len(names)
    names += [f"ProfilerStep#{i}" for i in range(iterations)]

    def emit(cat, start, dur, name, pid=None, parent=None, seq=None, addr=None,
             nbytes=None):
        n = len(start)

        def col(v):
            return np.full(n, NONE, np.int64) if v is None else np.asarray(v, np.int64)
        cols["cat"].append(np.full(n, cat, np.int8))
        cols["start"].append(np.asarray(start, np.int64))
        cols["dur"].append(np.asarray(dur, np.int64))
        cols["name"].append(np.asarray(name, np.int64) if np.ndim(name) else
                            np.full(n, name, np.int64))
        cols["pid"].append(col(pid))
        cols["parent"].append(col(parent))
        cols["seq"].append(col(seq))
        cols["addr"].append(col(addr))
        cols["nbytes"].append(col(nbytes))

    param = [hidden * hidden * 4, hidden * 4]
    act_size = hidden * 32 * 4
    L = leaves
    k = np.arange(L, dtype=np.int64)
    # address pools: one region per size class, recycled every iteration
    act_addr = 1 << 40 | (k * 4096)
    tmp_addr = 2 << 40 | ((k % 64) * 4096)
    grad_addr = [3 << 40 | (k * 2 * 4096), 3 << 40 | (k * 2 * 4096 + 4096)]
    state_addr = 4 << 40
    t = 0
    pid0 = 1
    seq0 = 1
    for it in range(iterations):
        step_start = t
        emit(UA, [t], [0], step_name0 + it)  # duration patched below
        step_idx = sum(len(c) for c in cols["start"]) - 1
        zs = t + 2
        emit(UA, [zs], [5], 8)
        if it > 0:  # zero_grad frees the previous iteration's gradients
            emit(IN, zs + 1 + k * 0, 0 * k, 9, addr=grad_addr[0], nbytes=-param[0] + 0 * k)
            emit(IN, zs + 2 + k * 0, 0 * k, 9, addr=grad_addr[1], nbytes=-param[1] + 0 * k)
        base = zs + 10
        # forward: model frame, per leaf: helper + layer frame, ops, instants
        span = 20
        fs = base + k * span
        model_pid = pid0
        emit(PF, [base - 1], [L * span + 2], 0, pid=[model_pid])
        helper_pid = pid0 + 1 + 2 * k
        leaf_pid = helper_pid + 1
        emit(PF, fs, 0 * k + 18, 1, pid=helper_pid, parent=model_pid + 0 * k)
        emit(PF, fs + 1, 0 * k + 16, leaf_name0 + k, pid=leaf_pid, parent=helper_pid)
        pid0 += 1 + 2 * L
        seqs = seq0 + k
        seq0 += L
        emit(OP, fs + 2, 0 * k + 12, 2, seq=seqs)                       # root
        emit(OP, fs + 3, 0 * k + 5, 3, seq=np.where(k % 3 == 0, seqs, -1))  # nested
        emit(OP, fs + 9, 0 * k + 4, 4, seq=0 * k - 1)                   # nested
        jitter = rng.integers(0, 2, L) * 512
        emit(IN, fs + 4, 0 * k, 9, addr=act_addr, nbytes=act_size + jitter)
        emit(IN, fs + 5, 0 * k, 9, addr=tmp_addr, nbytes=0 * k + act_size)
        emit(IN, fs + 8, 0 * k, 9, addr=tmp_addr, nbytes=0 * k - act_size)
        # backward, reverse order, outside the frames
        bbase = base + L * span + 10
        bs = bbase + (L - 1 - k) * span
        emit(OP, bs, 0 * k + 12, 5, seq=seqs)
        emit(OP, bs + 1, 0 * k + 3, 6, seq=0 * k - 1)
        emit(IN, bs + 2, 0 * k, 9, addr=grad_addr[0], nbytes=0 * k + param[0])
        emit(IN, bs + 3, 0 * k, 9, addr=grad_addr[1], nbytes=0 * k + param[1])
        emit(IN, bs + 6, 0 * k, 9, addr=act_addr, nbytes=-(act_size + jitter))
        # optimizer step: state in iteration 0, temporaries
        os_ = bbase + L * span + 10
        nst = min(L, 4096)
        if it == 0:
            ks = np.arange(nst, dtype=np.int64)
            emit(IN, os_ + 1 + ks, 0 * ks, 9, addr=state_addr + ks * 8192,
                 nbytes=0 * ks + param[0])
        emit(IN, [os_ + nst + 2, os_ + nst + 3], [0, 0], 9,
             addr=[5 << 40, 5 << 40], nbytes=[param[1], -param[1]])
        emit(UA, [os_], [nst + 5], 7)
        t = os_ + nst + 10
        _patch_step(cols, step_idx, t - step_start)  # the step spans it all
    cat = np.concatenate(cols["cat"])
    start = np.concatenate(cols["start"])
    dur = np.concatenate(cols["dur"])
    order = np.lexsort((np.arange(len(start)), start))  # stable by start
    ints = {"python_id": np.concatenate(cols["pid"])[order],
            "parent_id": np.concatenate(cols["parent"])[order],
            "sequence_number": np.concatenate(cols["seq"])[order],
            "addr": np.concatenate(cols["addr"])[order],
            "nbytes": np.concatenate(cols["nbytes"])[order],
            "total_allocated": np.full(len(start), NONE, np.int64),
            "total_reserved": np.full(len(start), NONE, np.int64)}
    seqv = ints["sequence_number"]
    ints["sequence_number"] = np.where(seqv < 0, NONE, seqv)
    name_ids = np.concatenate(cols["name"])[order]
    side = SidecarConfig(param_sizes=tuple(param), batch_bytes=(hidden * 32 * 4, 256),
                         optimizer_name="AdamW")
    return TraceBundle(category=cat[order], start=start[order] - start.min(),
                       duration=dur[order], ints=ints,
                       names=NameColumn(names, name_ids), metadata=side)


def _patch_step(cols, flat_index, dur):
    n = 0
    for arr in cols["dur"]:
        if flat_index < n + len(arr):
            arr[flat_index - n] = dur
            return
        n += len(arr)
