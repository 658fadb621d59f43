"""Batched estimation: many traces through analysis, link, orchestration and
replay in one pass each, device-resident between the stages.

The reference estimates one trace per call (PeakMemoryEstimator.estimate,
estimator.py:135-179: analyze -> build_sequence -> replay).  A batch-size
or config sweep (BASELINE configs C2 / C4) calls it once per trace.  Here
`build_sequences` hands the event columns of all traces to
`pm_pipeline_batch` (csrc/pipeline_batch.cuh) in one upload; the
orchestrated pm_req_t of every trace land in one device buffer in the layout
`pm_replay_batch` reads, and `PeakMemoryEstimator.estimate_many` replays
them as one batch and builds the reports -- byte-identical to calling
`estimate` on each bundle.

Host work per trace is what the reference also does on the host and is
tiny: the layer-name test (once per distinct name), marker typing and the
iteration / clone plan (orchestration.plan_sequence).  Errors surface per
trace in the reference's order (analysis, then sequence construction, then
replay); `estimate_many` raises the first failing trace's error, as a loop
over `estimate` would.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, _pipeline
from .analysis import LAYER_NAME_PREFIXES, ROLE_OF_CODE, _is_layer, extract_markers
from .errors import (CyclicParentLink, MissingBatchBytes, NoGradientBlocks,
                     NoIterationMarkers, NoIterations)
from .orchestration import plan_sequence
from .trace import NONE, EventCategory, TraceBundle


@dataclass
class _Trace:
    cols: dict
    plan: object = None
    error: BaseException | None = None  # the first host-side failure


def _is_layer_column(bundle: TraceBundle, idx: np.ndarray) -> np.ndarray:
    """The layer-name test (analysis.py:115-182) once per distinct name."""
    names = bundle.names
    if hasattr(names, "table_flags"):
        flag = names.table_flags(LAYER_NAME_PREFIXES)
        return flag[names.ids[idx]] if len(flag) else np.zeros(len(idx), bool)
    return np.fromiter((_is_layer(names[i], LAYER_NAME_PREFIXES)
                        for i in idx.tolist()), bool, len(idx))


# (column, category, bundle field) of the single host -> device upload;
# gathered straight into the pinned staging buffer
_GATHER = (("fn_pid", "fn", "python_id"), ("fn_par", "fn", "parent_id"),
           ("fn_start", "fn", "start"), ("fn_end", "fn", "end"),
           ("op_start", "op", "start"), ("op_end", "op", "end"),
           ("op_seq", "op", "sequence_number"), ("in_start", "in", "start"),
           ("in_addr", "in", "addr"), ("in_nbytes", "in", "nbytes"))
_CAT = {"fn": EventCategory.PYTHON_FUNCTION, "op": EventCategory.CPU_OP,
        "in": EventCategory.CPU_INSTANT_EVENT}


def _column(bundle: TraceBundle, field: str) -> np.ndarray:
    if field == "start":
        return bundle.start
    if field == "end":
        return bundle.end
    return bundle.ints[field]


def _trace(bundle: TraceBundle, iterations: int) -> _Trace:
    idx = {k: bundle.indices(c) for k, c in _CAT.items()}
    tr = _Trace({"idx": idx, "bundle": bundle})
    try:
        markers = extract_markers(bundle.by_category(EventCategory.USER_ANNOTATION))
    except NoIterationMarkers as e:
        tr.error = e
        return tr
    try:
        tr.plan = plan_sequence(markers, bundle.metadata, iterations)
    except (NoIterations, MissingBatchBytes) as e:
        tr.error = e
    return tr


class SequenceBatch:
    """Orchestrated request sequences of B traces, resident on the device.

    `d_reqs` (uint8 view of pm_req_t records) and `req_off` are exactly what
    pm_replay_batch takes; `errors[t]` is the exception build_sequence would
    raise for trace t (None if it succeeds; the requests of a failed trace
    are unspecified -- often none)."""

    def __init__(self, d_reqs, req_off, n_model, breakdown, errors, plans):
        self.d_reqs = d_reqs
        self.req_off = req_off
        self.n_model = n_model
        self.breakdown_codes = breakdown
        self.errors = errors
        self.plans = plans

    def __len__(self) -> int:
        return len(self.req_off) - 1

    def lengths(self) -> np.ndarray:
        return np.diff(self.req_off)

    def breakdown(self, t: int) -> dict[str, int]:
        """ALLOC bytes by role value of trace t (estimator.py:160-164)."""
        row = self.breakdown_codes[t]
        return {ROLE_OF_CODE[c].value: int(row[c]) for c in range(7) if row[c] > 0}

    def packed(self, t: int) -> np.ndarray:
        """Trace t's pm_req_t records on the host."""
        a, b = int(self.req_off[t]), int(self.req_off[t + 1])
        rs = _native.REQ_DTYPE.itemsize
        return self.d_reqs[a * rs:b * rs].cpu().numpy().view(_native.REQ_DTYPE).copy()


def build_sequences(bundles, iterations: int = 2, device: int | None = None,
                    views: bool = False) -> SequenceBatch:
    """orchestration.build_sequence(orchestration.analyze(b), iterations) for
    every bundle, in one pm_pipeline_batch call on `device` (default: the
    current CUDA device) and its current stream.  With views, the ordered
    request columns and the blocks' final roles / frees come back too, left
    on the device (`SequenceBatch.views`)."""
    import torch

    _native.require_device()
    if device is None:
        device = torch.cuda.current_device()
    with torch.cuda.device(device):
        return _build_sequences(bundles, iterations, device, views)


def _build_sequences(bundles, iterations, device, views) -> SequenceBatch:
    import torch

    bundles = list(bundles)
    B = len(bundles)
    if B == 0:
        raise ValueError("build_sequences needs at least one trace")
    traces = [_trace(b, iterations) for b in bundles]
    counts = {k: np.array([len(t.cols["idx"][k]) for t in traces], np.int64)
              for k in _CAT}

    def offs(counts):
        o = np.zeros(len(counts) + 1, np.int64)
        np.cumsum(counts, out=o[1:])
        return o

    fn_off, op_off, in_off = offs(counts["fn"]), offs(counts["op"]), offs(counts["in"])
    tot = {"fn": int(fn_off[-1]), "op": int(op_off[-1]), "in": int(in_off[-1])}
    toff = {"fn": fn_off, "op": op_off, "in": in_off}
    # one pinned host buffer (columns gathered straight into it) -> one upload
    total = sum(tot[k] for _, k, _ in _GATHER) + (tot["fn"] + 7) // 8
    dev = torch.device("cuda", device)
    h = torch.empty(max(total, 1), dtype=torch.int64, pin_memory=True)
    hv = h.numpy()
    pos = {}
    at = 0
    jobs = []
    for col, k, field in _GATHER:
        for t, tr in enumerate(traces):
            a, z = at + int(toff[k][t]), at + int(toff[k][t + 1])
            if z > a:
                jobs.append((_column(tr.cols["bundle"], field), tr.cols["idx"][k],
                             hv[a:z]))
        pos[col] = (at, tot[k])
        at += tot[k]
    # numpy's take releases the GIL: the column gathers run on host threads
    if len(jobs) > 1 and sum(len(j[1]) for j in jobs) > (1 << 20):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(jobs), 16)) as pool:
            list(pool.map(lambda j: np.take(j[0], j[1], out=j[2]), jobs))
    else:
        for src, idx, out in jobs:
            np.take(src, idx, out=out)
    # sequence numbers: None -> -1 (the kernels' "no sequence number")
    a, n = pos["op_seq"]
    if n:
        seqv = hv[a:a + n]
        seqv[seqv == NONE] = -1
    isl = hv[at:].view(np.uint8)
    for t, tr in enumerate(traces):
        a, z = int(fn_off[t]), int(fn_off[t + 1])
        if z > a:
            isl[a:z] = _is_layer_column(tr.cols["bundle"], tr.cols["idx"]["fn"])
    d = h.to(dev, non_blocking=True)
    base = d.data_ptr()

    desc = _pipeline.PipelineBatch()
    desc.n_traces = B
    keep = []  # host arrays the descriptor points at

    def host(a, dtype=np.int64):
        a = np.ascontiguousarray(a, dtype=dtype)
        keep.append(a)
        return a.ctypes.data if a.size else None

    desc.fn_off, desc.op_off, desc.in_off = host(fn_off), host(op_off), host(in_off)
    for c, _, _ in _GATHER:
        setattr(desc, c, base + 8 * pos[c][0] if pos[c][1] else None)
    desc.fn_is_layer = base + 8 * at if tot["fn"] else None

    # per-trace orchestration parameters (CSR)
    empty = ([], [], [])
    sp = [t.plan.spans if t.plan else empty for t in traces]
    pa = [t.plan.param_sizes if t.plan else [] for t in traces]
    wi = [t.plan.windows if t.plan else ([], []) for t in traces]
    zg = [t.plan.zg if t.plan else [] for t in traces]
    bt = [t.plan.batch if t.plan else ([], [], [], [], []) for t in traces]
    cat = lambda xs: np.concatenate([np.asarray(x, np.int64) for x in xs]) \
        if xs else np.zeros(0, np.int64)
    desc.span_off = host(offs([len(s[0]) for s in sp]))
    desc.span_start, desc.span_end, desc.span_iter = (
        host(cat([s[k] for s in sp])) for k in range(3))
    desc.param_off = host(offs([len(p) for p in pa]))
    desc.param_sizes = host(cat(pa))
    desc.win_off = host(offs([len(w[0]) for w in wi]))
    desc.win_start, desc.win_end = host(cat([w[0] for w in wi])), host(cat([w[1] for w in wi]))
    desc.zg_off = host(offs([len(z) for z in zg]))
    desc.zg = host(cat(zg))
    clones = np.array([t.plan.clones if t.plan else 0 for t in traces], np.int32)
    desc.clones = host(clones, np.int32)
    desc.tpl_start = host([t.plan.tpl[0] if t.plan else 0 for t in traces])
    desc.tpl_end = host([t.plan.tpl[1] if t.plan else 0 for t in traces])
    desc.shift = host([t.plan.shift if t.plan else 0 for t in traces])
    desc.bat_off = host(offs([len(b[0]) for b in bt]))
    desc.bat_vts, desc.bat_size = host(cat([b[0] for b in bt])), host(cat([b[1] for b in bt]))
    desc.bat_kind = host(cat([b[2] for b in bt]), np.int32)
    desc.bat_it, desc.bat_j = host(cat([b[3] for b in bt])), host(cat([b[4] for b in bt]))
    desc.skip = host([1 if t.error is not None else 0 for t in traces], np.int32)

    # requests per trace <= model (<= blocks) + batch + 2 blocks (1 + clones)
    bat_counts = np.array([len(b[0]) for b in bt], np.int64)
    cap = int((counts["in"] * (3 + 2 * clones.astype(np.int64)) + bat_counts).sum()) + 16
    rs = _native.REQ_DTYPE.itemsize
    d_reqs = torch.empty(cap * rs, dtype=torch.uint8, device=dev)
    req_off, status, n_model, bd, vw = _pipeline.pipeline_batch(
        desc, d_reqs.data_ptr(), cap, B,
        fb_cap=int(counts["in"].sum()) if views else None)
    del d, h  # the call synchronised its stream: the upload is consumed
    errors: list[BaseException | None] = []
    for t, tr in enumerate(traces):
        st = int(status[t])
        if st == _pipeline.PM_ERR_CYCLIC_PARENT:
            errors.append(CyclicParentLink("parent chain revisits a python id"))
        elif tr.error is not None:
            errors.append(tr.error)
        elif st == -1:
            errors.append(NoGradientBlocks("no backward-retained blocks in trace"))
        elif not tr.plan.has_batch_bytes:
            errors.append(MissingBatchBytes("sidecar provides no batch tensor sizes"))
        elif st != 0:
            errors.append(RuntimeError(f"pm_pipeline_batch: trace {t} status {st}"))
        else:
            errors.append(None)
    sb = SequenceBatch(d_reqs, req_off, n_model, bd, errors, [t.plan for t in traces])
    sb.views = vw
    return sb


__all__ = ["SequenceBatch", "build_sequences"]
