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

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _pipeline
from .analysis import (AnnotationMarker, BlockRole, LayerNode, MarkerKind,
                       MemoryBlock, OperatorNode, ROLE_OF_CODE,
                       blocks_from_link, build_layer_tree, extract_markers,
                       roots_from_link)
from .errors import MissingBatchBytes, NoGradientBlocks, NoIterations
from .linking import LayerMemoryProfile, non_wrapper_layers, profiles_from_link
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


@dataclass
class RequestSequence:
    """orchestration.py:70-87, plus the packed replay records."""

    requests: list[MemoryRequest]
    iteration_boundaries: list[int]
    phase_tags: dict
    packed: np.ndarray | None = field(default=None, repr=False, compare=False)

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


@dataclass
class AnalyzedTrace:
    """orchestration.py:90-104"""

    bundle: TraceBundle
    layer_tree: LayerNode
    operator_roots: list[OperatorNode]
    markers: list[AnnotationMarker]
    blocks: list[MemoryBlock]
    profiles: dict
    # device-side link result (block roles incl. the gradient tags)
    _link: object = field(default=None, repr=False, compare=False)

    def steps(self) -> list[AnnotationMarker]:
        return sorted((m for m in self.markers
                       if m.kind is MarkerKind.PROFILER_STEP),
                      key=lambda m: m.iteration_index)


def analyze(bundle: TraceBundle) -> AnalyzedTrace:
    """Build every structural view and link them (orchestration.py:107-116)."""
    tree = build_layer_tree(bundle.by_category(EventCategory.PYTHON_FUNCTION))
    ops = bundle.indices(EventCategory.CPU_OP)
    inst = bundle.indices(EventCategory.CPU_INSTANT_EVENT)
    markers = extract_markers(bundle.by_category(EventCategory.USER_ANNOTATION))
    leaves = non_wrapper_layers(tree)
    seq = bundle.ints["sequence_number"][ops]
    seq = np.where(seq == NONE, -1, seq)
    lk = _pipeline.link(bundle.start[ops], bundle.end[ops], seq,
                        bundle.start[inst], bundle.ints["addr"][inst],
                        bundle.ints["nbytes"][inst],
                        np.array([n.start_ts for n in leaves], np.int64),
                        np.array([n.end_ts for n in leaves], np.int64))
    op_names = [bundle.names[i] for i in ops.tolist()]
    roots = roots_from_link(op_names, None, None, lk)
    blocks = blocks_from_link(bundle.ints["addr"][inst], lk)
    profiles = profiles_from_link(leaves, roots, blocks, lk)
    return AnalyzedTrace(bundle=bundle, layer_tree=tree, operator_roots=roots,
                         markers=markers, blocks=blocks, profiles=profiles,
                         _link=lk)


def _block_id(tag: int, a: int, b: int):
    if tag == 0:
        return f"model:{a}"
    if tag == 1:
        return f"batch:{a}:{b}"
    if tag == 2:
        return a
    return f"clone{a}:{b}"


def build_sequence(analyzed: AnalyzedTrace, iterations: int = 2,
                   ) -> RequestSequence:
    """Assemble the replayable request sequence (orchestration.py:237-399)."""
    if iterations < 1:
        raise NoIterations(f"iterations must be >= 1, got {iterations}")
    sidecar = analyzed.bundle.metadata
    if sidecar is None:
        raise MissingBatchBytes(
            "orchestration requires a sidecar (param_sizes, batch_bytes)")
    steps = analyzed.steps()
    if not steps:
        raise NoIterations("trace has no iteration markers")
    lk = analyzed._link
    n_trace = len(steps)
    include = min(iterations, n_trace)
    clones = iterations - include
    windows = []
    for k in range(include):
        start = steps[k].start_ts
        end = steps[k + 1].start_ts if k + 1 < n_trace else steps[k].end_ts
        windows.append((start, end))

    spans = [m for m in analyzed.markers if m.kind is MarkerKind.OPTIMIZER_STEP]
    tpl = windows[-1]
    width = tpl[1] - tpl[0]
    clone_markers = []
    if clones:
        tpl_markers = [m for m in analyzed.markers
                       if m.iteration_index == include - 1
                       and tpl[0] <= m.start_ts < tpl[1]]
        for c in range(1, clones + 1):
            for m in tpl_markers:
                clone_markers.append(AnnotationMarker(
                    m.kind, m.start_ts + width * c, m.end_ts + width * c,
                    include - 1 + c))
    all_markers = list(analyzed.markers) + clone_markers
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

    blocks = analyzed.blocks
    nb = len(blocks)
    role_codes = lk.b_role if nb else np.zeros(0, np.int32)
    o = _pipeline.orchestrate(
        lk.b_alloc, lk.b_size, lk.b_free, role_codes,
        ([m.start_ts for m in spans], [m.end_ts for m in spans],
         [m.iteration_index for m in spans]),
        sorted(set(sidecar.param_sizes)),
        ([w[0] for w in windows], [w[1] for w in windows]), zg, clones,
        tpl if clones else (0, 0), width,
        (bv, bs, bk, bi, bj))
    if o.n < 0:
        raise NoGradientBlocks("no backward-retained blocks in trace")
    if not sidecar.batch_bytes:
        raise MissingBatchBytes("sidecar provides no batch tensor sizes")

    # the reference mutates the analyzed blocks in place
    for blk, rc, fr in zip(blocks, o.fb_role.tolist(), o.fb_free.tolist()):
        blk.role = ROLE_OF_CODE[rc]
        blk.free_time = None if fr == NONE else fr

    requests = []
    phase_tags: dict = {}
    kinds = (RequestKind.ALLOC, RequestKind.FREE)
    for i in range(o.n_model):
        phase_tags[f"model:{i}"] = BlockRole.MODEL
    for it, j in zip(bi[::2], bj[::2]):
        phase_tags[f"batch:{it}:{j}"] = BlockRole.BATCH
    # chosen blocks then clones, in raw (emission) order
    raw_order = np.argsort(o.raw, kind="stable")
    tags, aa, bb, roles, kk = (o.tag.tolist(), o.a.tolist(), o.b.tolist(),
                               o.role.tolist(), o.kind.tolist())
    for i in raw_order.tolist():
        if tags[i] >= 2 and kk[i] == 0:
            phase_tags[_block_id(tags[i], aa[i], bb[i])] = ROLE_OF_CODE[roles[i]]
    for seq_no, (t, a, b, kind, size, vts) in enumerate(zip(
            tags, aa, bb, kk, o.size.tolist(), o.vts.tolist())):
        requests.append(MemoryRequest(seq_no=seq_no, kind=kinds[kind],
                                      block_id=_block_id(t, a, b), size=size,
                                      virtual_ts=vts))
    boundaries = [w[0] for w in windows]
    end = windows[-1][1]
    if clones:
        for c in range(1, clones + 1):
            boundaries.append(windows[-1][0] + width * c)
        end = windows[-1][0] + width * (clones + 1)
    boundaries.append(end)
    return RequestSequence(requests=requests, iteration_boundaries=boundaries,
                           phase_tags=phase_tags, packed=o.packed)


__all__ = ["AnalyzedTrace", "MemoryRequest", "RequestKind", "RequestSequence",
           "analyze", "build_sequence", "LayerMemoryProfile"]
