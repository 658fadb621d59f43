"""Sequence orchestration, mirroring peakmem.orchestration
(pkg/src/peakmem/orchestration.py).

`analyze` runs the layer tree and markers on the host and every per-event /
per-op / per-block stage in one `pm_link` call; `build_sequence` derives the
iteration windows, spans and cloned markers on the host (a handful of
markers) and runs the per-block state / drop / clone / gradient-lifetime
rewrites, the model-load and request emission and the (virtual_ts, rank,
idx) total order in one `pm_orchestrate` call.  The result carries the
packed replay records so the estimator feeds the replay kernel directly.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _pipeline
from .analysis import (AnnotationMarker, BlockRole, LayerNode,
                       LayerTreeColumns, MarkerKind, MemoryBlock, OperatorNode,
                       ROLE_OF_CODE, blocks_from_link, extract_markers,
                       roots_from_link)
from .errors import MissingBatchBytes, NoGradientBlocks, NoIterations
from .linking import LayerMemoryProfile, profiles_from_link
from .trace import EventCategory, NONE, TraceBundle


class RequestKind(Enum):
    ALLOC = "alloc"
    FREE = "free"


@dataclass(frozen=True)
class MemoryRequest:
    """orchestration.py:55-67"""

    seq_no: int
    kind: RequestKind
    block_id: int | str
    size: int
    virtual_ts: int
    stream: int = 0

    def to_json_dict(self) -> dict:
        return {"seq_no": self.seq_no, "kind": self.kind.value,
                "block_id": self.block_id, "size": self.size,
                "virtual_ts": self.virtual_ts, "stream": self.stream}


class RequestSequence:
    """orchestration.py:70-87.  Built by build_sequence from the device's
    ordered arrays; `requests` and `phase_tags` materialise on first use
    (the estimator reads only the arrays and the packed replay records)."""

    def __init__(self, requests=None, iteration_boundaries=None,
                 phase_tags=None, packed=None, arrays=None):
        self._requests = requests
        self.iteration_boundaries = list(iteration_boundaries or [])
        self._phase_tags = phase_tags
        self._packed = packed
        self._packed_src = None  # a batch.SequenceBatch holding it on the device
        self._breakdown = None
        self._arrays = arrays

    @property
    def packed(self):
        """The packed pm_req_t replay records (host)."""
        if self._packed is None and self._packed_src is not None:
            self._packed = self._packed_src.packed(0)
            self._packed_src = None
        return self._packed

    @packed.setter
    def packed(self, value):
        self._packed = value
        self._packed_src = None

    def __len__(self) -> int:
        if self._requests is not None:
            return len(self._requests)
        return int(self._arrays["n"])

    @property
    def requests(self) -> list[MemoryRequest]:
        if self._requests is None:
            a = self._arrays
            kinds = (RequestKind.ALLOC, RequestKind.FREE)
            self._requests = [
                MemoryRequest(seq_no=i, kind=kinds[k], block_id=_block_id(t, x, y),
                              size=sz, virtual_ts=v)
                for i, (t, x, y, k, sz, v) in enumerate(zip(
                    a["tag"].tolist(), a["a"].tolist(), a["b"].tolist(),
                    a["kind"].tolist(), a["size"].tolist(), a["vts"].tolist()))]
        return self._requests

    @property
    def phase_tags(self) -> dict:
        if self._phase_tags is None:
            a = self._arrays
            tags: dict = {}
            for i in range(a["n_model"]):
                tags[f"model:{i}"] = BlockRole.MODEL
            for it, j in a["batch_ids"]:
                tags[f"batch:{it}:{j}"] = BlockRole.BATCH
            order = np.argsort(a["raw"], kind="stable")
            tg, x, y, rl, k = (a["tag"][order], a["a"][order], a["b"][order],
                               a["role"][order], a["kind"][order])
            sel = (tg >= 2) & (k == 0)
            for t, xx, yy, r in zip(tg[sel].tolist(), x[sel].tolist(),
                                    y[sel].tolist(), rl[sel].tolist()):
                tags[_block_id(t, xx, yy)] = ROLE_OF_CODE[r]
            self._phase_tags = tags
        return self._phase_tags

    def breakdown(self) -> dict[str, int]:
        """Sum of ALLOC sizes per role value (estimator.py:160-164)."""
        if self._breakdown is not None:
            return dict(self._breakdown)
        if self._arrays is None:
            out: dict[str, int] = {}
            for r in self.requests:
                if r.kind is RequestKind.ALLOC:
                    role = self.phase_tags[r.block_id].value
                    out[role] = out.get(role, 0) + r.size
            return out
        a = self._arrays
        alloc = a["kind"] == 0
        roles = a["role"][alloc]
        sizes = a["size"][alloc]
        out = {}
        for code in np.unique(roles).tolist():
            out[ROLE_OF_CODE[code].value] = int(sizes[roles == code].sum())
        return out

    def to_json_dict(self) -> dict:
        return {
            "requests": [r.to_json_dict() for r in self.requests],
            "iteration_boundaries": list(self.iteration_boundaries),
            "phase_tags": {str(k): v.value for k, v in self.phase_tags.items()},
        }

    def replay_records(self) -> list[dict]:
        return [{"seq_no": r.seq_no, "kind": r.kind.value,
                 "block_id": r.block_id, "size": r.size, "stream": r.stream}
                for r in self.requests]


class AnalyzedTrace:
    """orchestration.py:90-104.  Structural views of one bundle; the object
    views (layer_tree, operator_roots, blocks, profiles) materialise from
    the device's columnar link result on first access."""

    def __init__(self, bundle, tree_cols, markers, link, op_idx):
        self.bundle = bundle
        self.markers = markers
        self._tree = tree_cols
        self._link_data = link  # None until a view needs it
        self._ops = op_idx
        self._objects = None
        self._final = None  # (roles, frees) of the last build_sequence

    @property
    def _link(self):
        """pm_link's columnar result, computed on first use (the object
        views need it; build_sequence alone runs the batched pipeline)."""
        if self._link_data is None:
            self._link_data = _link_columns(self.bundle, self._tree, self._ops)
        return self._link_data

    def _materialise(self):
        if self._objects is None:
            root, leaves = self._tree.tree()
            names = self.bundle.names
            op_names = [names[i] for i in self._ops.tolist()]
            roots = roots_from_link(op_names, None, None, self._link)
            inst = self.bundle.indices(EventCategory.CPU_INSTANT_EVENT)
            blocks = blocks_from_link(self.bundle.ints["addr"][inst], self._link)
            profiles = profiles_from_link(leaves, roots, blocks, self._link)
            self._objects = (root, roots, blocks, profiles)
            if self._final is not None:
                self._apply_final()
        return self._objects

    @property
    def layer_tree(self) -> LayerNode:
        return self._materialise()[0]

    @property
    def operator_roots(self) -> list[OperatorNode]:
        return self._materialise()[1]

    @property
    def blocks(self) -> list[MemoryBlock]:
        return self._materialise()[2]

    @property
    def profiles(self) -> dict:
        return self._materialise()[3]

    def _apply_final(self):
        """build_sequence mutates the analyzed blocks in place, like the
        reference (orchestration.py:222-223, 197)."""
        roles, frees = self._final if isinstance(self._final, tuple) else self._final.get()
        for blk, rc, fr in zip(self._objects[2], roles.tolist(), frees.tolist()):
            blk.role = ROLE_OF_CODE[rc]
            blk.free_time = None if fr == NONE else fr

    def steps(self) -> list[AnnotationMarker]:
        return sorted((m for m in self.markers
                       if m.kind is MarkerKind.PROFILER_STEP),
                      key=lambda m: m.iteration_index)


def _link_columns(bundle: TraceBundle, tree, ops):
    inst = bundle.indices(EventCategory.CPU_INSTANT_EVENT)
    seq = bundle.ints["sequence_number"][ops]
    seq = np.where(seq == NONE, -1, seq)
    return _pipeline.link(bundle.start[ops], bundle.end[ops], seq,
                          bundle.start[inst], bundle.ints["addr"][inst],
                          bundle.ints["nbytes"][inst], tree.leaf_start,
                          tree.leaf_end)


def analyze(bundle: TraceBundle) -> AnalyzedTrace:
    """Build every structural view and link them (orchestration.py:107-116).

    The layer tree (CyclicParentLink) and the markers (NoIterationMarkers)
    are built here, in the reference's order; the operator / block link is
    computed when a view needs it -- build_sequence on its own takes the
    batched device pipeline, which links on the device without a round trip."""
    tree = LayerTreeColumns(bundle)
    ops = bundle.indices(EventCategory.CPU_OP)
    markers = extract_markers(bundle.by_category(EventCategory.USER_ANNOTATION))
    return AnalyzedTrace(bundle, tree, markers, None, ops)


def _block_id(tag: int, a: int, b: int):
    if tag == 0:
        return f"model:{a}"
    if tag == 1:
        return f"batch:{a}:{b}"
    if tag == 2:
        return a
    return f"clone{a}:{b}"


class _Plan:
    """The host half of build_sequence for one trace: iteration windows,
    optimizer spans, cloned markers, zero-grad marks and the batch requests
    (a handful of markers; orchestration.py:237-336)."""


def plan_sequence(markers, sidecar, iterations: int) -> _Plan:
    """Raises what build_sequence raises before touching the blocks."""
    if iterations < 1:
        raise NoIterations(f"iterations must be >= 1, got {iterations}")
    if sidecar is None:
        raise MissingBatchBytes(
            "orchestration requires a sidecar (param_sizes, batch_bytes)")
    steps = sorted((m for m in markers if m.kind is MarkerKind.PROFILER_STEP),
                   key=lambda m: m.iteration_index)
    if not steps:
        raise NoIterations("trace has no iteration markers")
    n_trace = len(steps)
    include = min(iterations, n_trace)
    clones = iterations - include
    windows = []
    for k in range(include):
        start = steps[k].start_ts
        end = steps[k + 1].start_ts if k + 1 < n_trace else steps[k].end_ts
        windows.append((start, end))

    spans = [m for m in markers if m.kind is MarkerKind.OPTIMIZER_STEP]
    tpl = windows[-1]
    width = tpl[1] - tpl[0]
    clone_markers = []
    if clones:
        tpl_markers = [m for m in markers
                       if m.iteration_index == include - 1
                       and tpl[0] <= m.start_ts < tpl[1]]
        for c in range(1, clones + 1):
            for m in tpl_markers:
                clone_markers.append(AnnotationMarker(
                    m.kind, m.start_ts + width * c, m.end_ts + width * c,
                    include - 1 + c))
    all_markers = list(markers) + clone_markers
    zg = sorted(m.start_ts for m in all_markers if m.kind is MarkerKind.ZERO_GRAD)
    step_markers = sorted((m for m in all_markers
                           if m.kind is MarkerKind.PROFILER_STEP
                           and m.iteration_index < iterations),
                          key=lambda m: m.iteration_index)
    bv, bs, bk, bi, bj = [], [], [], [], []
    for step in step_markers:
        for j, size in enumerate(sidecar.batch_bytes):
            bv += [step.start_ts, step.end_ts]
            bs += [size, size]
            bk += [0, 1]
            bi += [step.iteration_index] * 2
            bj += [j, j]
    p = _Plan()
    p.spans = ([m.start_ts for m in spans], [m.end_ts for m in spans],
               [m.iteration_index for m in spans])
    p.param_sizes = sorted(set(sidecar.param_sizes))
    p.windows = ([w[0] for w in windows], [w[1] for w in windows])
    p.zg = zg
    p.clones = clones
    p.tpl = tpl if clones else (0, 0)
    p.shift = width
    p.batch = (bv, bs, bk, bi, bj)
    p.batch_ids = list(zip(bi[::2], bj[::2]))
    p.has_batch_bytes = bool(sidecar.batch_bytes)
    boundaries = [w[0] for w in windows]
    end = windows[-1][1]
    if clones:
        for c in range(1, clones + 1):
            boundaries.append(windows[-1][0] + width * c)
        end = windows[-1][0] + width * (clones + 1)
    boundaries.append(end)
    p.boundaries = boundaries
    return p


def build_sequence(analyzed: AnalyzedTrace, iterations: int = 2,
                   ) -> RequestSequence:
    """Assemble the replayable request sequence (orchestration.py:237-399)."""
    plan = plan_sequence(analyzed.markers, analyzed.bundle.metadata, iterations)
    if analyzed._link_data is None:
        return _build_batched(analyzed, plan, iterations)
    lk = analyzed._link
    nb = int(lk.n_blocks)
    role_codes = lk.b_role if nb else np.zeros(0, np.int32)
    o = _pipeline.orchestrate(
        lk.b_alloc, lk.b_size, lk.b_free, role_codes, plan.spans,
        plan.param_sizes, plan.windows, plan.zg, plan.clones, plan.tpl,
        plan.shift, plan.batch)
    if o.n < 0:
        raise NoGradientBlocks("no backward-retained blocks in trace")
    if not plan.has_batch_bytes:
        raise MissingBatchBytes("sidecar provides no batch tensor sizes")

    # the reference mutates the analyzed blocks in place
    analyzed._final = (o.fb_role, o.fb_free)
    if analyzed._objects is not None:
        analyzed._apply_final()
    arrays = {"n": o.n, "n_model": o.n_model, "kind": o.kind, "size": o.size,
              "vts": o.vts, "tag": o.tag, "a": o.a, "b": o.b, "role": o.role,
              "raw": o.raw, "batch_ids": plan.batch_ids}
    return RequestSequence(iteration_boundaries=plan.boundaries, packed=o.packed,
                           arrays=arrays)


class _DeviceArrays(dict):
    """RequestSequence arrays left on the device by pm_pipeline_batch's
    views: read back on the first access of a column (the estimator needs
    none of them)."""

    def __init__(self, host: dict, dev: dict, n: int):
        super().__init__(host)
        self._dev = dev
        self._n = n

    def __missing__(self, key):
        if key not in self._dev:
            raise KeyError(key)
        val = self._dev[key][:self._n].cpu().numpy()
        self[key] = val
        return val


class _LazyFinal:
    """analyzed._final of the batched path: (roles, frees), read back only
    if the analyzed trace's block views are materialised."""

    def __init__(self, dev: dict, nb: int):
        self._dev, self._nb = dev, nb
        self._val = None

    def get(self):
        if self._val is None:
            self._val = (self._dev["fb_role"][:self._nb].cpu().numpy(),
                         self._dev["fb_free"][:self._nb].cpu().numpy())
        return self._val


def _native_req_bytes() -> int:
    from ._native import REQ_DTYPE
    return REQ_DTYPE.itemsize


def _build_batched(analyzed: AnalyzedTrace, plan, iterations: int) -> RequestSequence:
    """build_sequence through pm_pipeline_batch (B = 1) with its views:
    link, orchestration and the total order on the device in one call; the
    views stay on the device until something reads them."""
    from .batch import build_sequences
    sb = build_sequences([analyzed.bundle], iterations, views=True)
    if sb.errors[0] is not None:
        raise sb.errors[0]
    n = int(sb.req_off[1])
    nb = int(sb.views["blk_off"][1])
    # keep right-sized device copies only (the call's buffers are sized for
    # the worst case)
    v = {f: (t[:nb] if f.startswith("fb_") else t[:n]).clone()
         for f, t in sb.views.items() if f != "blk_off"}
    rs = _native_req_bytes()
    sb.d_reqs = sb.d_reqs[:n * rs].clone()
    sb.views = None
    analyzed._final = _LazyFinal(v, nb)
    if analyzed._objects is not None:
        analyzed._apply_final()
    arrays = _DeviceArrays({"n": n, "n_model": int(sb.n_model[0]),
                            "batch_ids": plan.batch_ids}, v, n)
    seq = RequestSequence(iteration_boundaries=plan.boundaries, packed=None,
                          arrays=arrays)
    seq._packed_src = sb
    seq._breakdown = sb.breakdown(0)
    return seq


__all__ = ["AnalyzedTrace", "MemoryRequest", "RequestKind", "RequestSequence",
           "analyze", "build_sequence", "plan_sequence", "LayerMemoryProfile"]
