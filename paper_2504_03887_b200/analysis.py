"""Event analysis, mirroring peakmem.analysis (pkg/src/peakmem/analysis.py).

Host: the layer tree (string-typed module frames, parent-chain walk,
analysis.py:115-182) and marker typing (analysis.py:214-249) -- a few hundred
nodes.  Device: operator roots (analysis.py:185-211) and alloc/free grouping
(analysis.py:252-294) run in `pm_link` (csrc/pipeline.cu); the list-based
functions here are thin adapters onto those kernels for API parity.
"""

from __future__ import annotations

import logging
from bisect import bisect_right
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _pipeline
from .errors import CyclicParentLink, NoIterationMarkers
from .trace import EventCategory, TraceEvent

logger = logging.getLogger(__name__)

LAYER_NAME_PREFIXES = ("nn.Module: ",)


@dataclass(eq=False)
class LayerNode:
    """A module-call frame (analysis.py:32-50); identity semantics."""

    name: str
    start_ts: int
    end_ts: int
    children: list["LayerNode"] = field(default_factory=list)
    is_wrapper: bool = False
    event_id: int = -1

    def walk(self):
        stack = [self]
        while stack:
            node = stack.pop()
            yield node
            stack.extend(reversed(node.children))


@dataclass(eq=False)
class OperatorNode:
    """A top-level operator interval (analysis.py:53-68)."""

    name: str
    start_ts: int
    end_ts: int
    sequence_numbers: set[int] = field(default_factory=set)
    is_root: bool = True

    def contains_ts(self, ts: int) -> bool:
        return self.start_ts <= ts < self.end_ts


class MarkerKind(Enum):
    PROFILER_STEP = "profiler_step"
    ZERO_GRAD = "zero_grad"
    OPTIMIZER_STEP = "optimizer_step"


@dataclass(frozen=True)
class AnnotationMarker:
    kind: MarkerKind
    start_ts: int
    end_ts: int
    iteration_index: int


class BlockRole(Enum):
    UNCLASSIFIED = "unclassified"
    MODEL = "model"
    BATCH = "batch"
    GRADIENT = "gradient"
    OPTIMIZER_STATE = "optimizer_state"
    TEMPORARY = "temporary"
    RETAINED = "retained"


# role codes used by the kernels (csrc/pipeline.cu enum Role)
ROLE_OF_CODE = {0: BlockRole.UNCLASSIFIED, 1: BlockRole.MODEL,
                2: BlockRole.BATCH, 3: BlockRole.GRADIENT,
                4: BlockRole.OPTIMIZER_STATE, 5: BlockRole.TEMPORARY,
                6: BlockRole.RETAINED}
CODE_OF_ROLE = {v: k for k, v in ROLE_OF_CODE.items()}


@dataclass
class MemoryBlock:
    """One alloc/free lifetime (analysis.py:95-108)."""

    block_id: int
    addr: int
    size: int
    alloc_time: int
    free_time: int | None = None
    role: BlockRole = BlockRole.UNCLASSIFIED

    @property
    def permanent(self) -> bool:
        return self.free_time is None


def _is_layer(name: str, prefixes) -> bool:
    return name.startswith(prefixes)


def build_layer_tree(functions: list[TraceEvent],
                     layer_prefixes: tuple[str, ...] = LAYER_NAME_PREFIXES,
                     ) -> LayerNode:
    """Module-call frames as a tree (analysis.py:115-182): non-layer frames
    collapse, each layer hangs under its nearest layer ancestor through the
    python parent chain (first python id wins, cycles raise) -- the walk,
    child order and pre-order on the device (pm_layer_tree)."""
    for e in functions:
        if e.category is not EventCategory.PYTHON_FUNCTION:
            raise ValueError(f"not a python_function event: {e.name!r}")
    seen: set[int] = set()
    for e in functions:
        if e.python_id is not None:
            if e.python_id in seen:
                logger.warning("duplicate python id %s (%r); keeping the first",
                               e.python_id, e.name)
            seen.add(e.python_id)
    none = _pipeline.NONE
    is_layer = np.array([_is_layer(e.name, layer_prefixes) for e in functions],
                        bool)
    node_parent, order, off, _walk = _pipeline.layer_tree(
        [none if e.python_id is None else e.python_id for e in functions],
        [none if e.parent_id is None else e.parent_id for e in functions],
        is_layer, [e.start_ts for e in functions],
        [e.event_id for e in functions])
    layers = [e for e, f in zip(functions, is_layer.tolist()) if f]
    nodes = []
    for e in layers:
        shown = e.name
        for prefix in layer_prefixes:
            if shown.startswith(prefix):
                shown = shown[len(prefix):]
                break
        nodes.append(LayerNode(name=shown, start_ts=e.start_ts, end_ts=e.end_ts,
                               event_id=e.event_id))
    root = LayerNode(name="<root>", start_ts=0, end_ts=0, is_wrapper=True)
    o = order.tolist()
    off = off.tolist()
    root.children = [nodes[v] for v in o[off[0]:off[1]]]
    for k, node in enumerate(nodes):
        node.children = [nodes[v] for v in o[off[k + 1]:off[k + 2]]]
        node.is_wrapper = bool(node.children)
    if root.children:
        root.start_ts = min(c.start_ts for c in root.children)
        root.end_ts = max(c.end_ts for c in root.children)
    return root


def _marker_kind(name: str) -> MarkerKind | None:
    if name.startswith("ProfilerStep"):
        return MarkerKind.PROFILER_STEP
    if "zero_grad" in name:
        return MarkerKind.ZERO_GRAD
    if name.startswith("Optimizer.step") or name.endswith(".step"):
        return MarkerKind.OPTIMIZER_STEP
    return None


def extract_markers(annotations: list[TraceEvent]) -> list[AnnotationMarker]:
    """Typed iteration markers (analysis.py:214-249)."""
    for e in annotations:
        if e.category is not EventCategory.USER_ANNOTATION:
            raise ValueError(f"not a user_annotation event: {e.name!r}")
    typed = [(e, _marker_kind(e.name)) for e in annotations]
    steps = sorted((e for e, k in typed if k is MarkerKind.PROFILER_STEP),
                   key=lambda e: (e.start_ts, e.event_id))
    if not steps:
        raise NoIterationMarkers("no profiler-step annotations in trace")
    starts = [e.start_ts for e in steps]
    out = [AnnotationMarker(MarkerKind.PROFILER_STEP, e.start_ts, e.end_ts, i)
           for i, e in enumerate(steps)]
    for e, kind in typed:
        if kind in (MarkerKind.ZERO_GRAD, MarkerKind.OPTIMIZER_STEP):
            it = max(0, bisect_right(starts, e.start_ts) - 1)
            out.append(AnnotationMarker(kind, e.start_ts, e.end_ts, it))
    out.sort(key=lambda m: (m.start_ts, m.kind.value))
    return out


def roots_from_link(names: list[str], op_start, op_end, link) -> list[OperatorNode]:
    """OperatorNode objects from pm_link's root columns."""
    roots = []
    off = link.root_seq_off.tolist()
    seqs = link.root_seq.tolist()
    for r, (op, s, e) in enumerate(zip(link.root_op.tolist(),
                                       link.root_start.tolist(),
                                       link.root_end.tolist())):
        roots.append(OperatorNode(name=names[op], start_ts=s, end_ts=e,
                                  sequence_numbers=set(seqs[off[r]:off[r + 1]])))
    return roots


def blocks_from_link(addr, link) -> list[MemoryBlock]:
    """MemoryBlock objects (link-time roles: gradients show as retained)."""
    out = []
    for b, (i, t, sz, fr, rc) in enumerate(zip(
            link.b_inst.tolist(), link.b_alloc.tolist(), link.b_size.tolist(),
            link.b_free.tolist(), link.b_role.tolist())):
        role = ROLE_OF_CODE[6 if rc == 3 else rc]
        out.append(MemoryBlock(block_id=b, addr=int(addr[i]), size=sz,
                               alloc_time=t, free_time=None if fr == _pipeline.NONE else fr,
                               role=role))
    return out


def build_operator_roots(ops: list[TraceEvent]) -> list[OperatorNode]:
    """Top-level operator forest (analysis.py:185-211), on the GPU."""
    for e in ops:
        if e.category is not EventCategory.CPU_OP:
            raise ValueError(f"not a cpu_op event: {e.name!r}")
    if not ops:
        return []
    # event ids order the ops exactly as the reference's tie-break does
    ops = sorted(ops, key=lambda e: e.event_id)
    st = np.array([e.start_ts for e in ops], np.int64)
    en = np.array([e.end_ts for e in ops], np.int64)
    sq = np.array([-1 if e.sequence_number is None else e.sequence_number
                   for e in ops], np.int64)
    z = np.zeros(0, np.int64)
    link = _pipeline.link(st, en, sq, z, z, z, z, z)
    return roots_from_link([e.name for e in ops], st, en, link)


def group_memory_events(instants: list[TraceEvent]) -> list[MemoryBlock]:
    """Alloc/free pairing by address recurrence (analysis.py:252-294), on the
    GPU."""
    for e in instants:
        if e.category is not EventCategory.CPU_INSTANT_EVENT:
            raise ValueError(f"not a cpu_instant_event: {e.name!r}")
    if not instants:
        return []
    ev = sorted(instants, key=lambda e: (e.start_ts, e.event_id))
    st = np.array([e.start_ts for e in ev], np.int64)
    ad = np.array([e.addr for e in ev], np.int64)
    nb = np.array([e.nbytes for e in ev], np.int64)
    z = np.zeros(0, np.int64)
    link = _pipeline.link(z, z, z, st, ad, nb, z, z)
    return blocks_from_link(ad, link)


class LayerTreeColumns:
    """The layer tree of analysis.py:115-182 computed from bundle columns.

    Nearest-layer ancestors, the (start, event_id) child order and the
    pre-order walk come from `pm_layer_tree` on the device (first python id
    wins; a chain that returns to its own id or never terminates raises
    CyclicParentLink, as the reference's seen-set does); the walk gives the
    non-wrapper layers (leaves) the link kernels consume.  LayerNode objects
    are built only on demand (`tree()`).
    """

    def __init__(self, bundle):
        from .trace import EventCategory as EC
        idx = bundle.indices(EC.PYTHON_FUNCTION)
        self.bundle = bundle
        pid = bundle.ints["python_id"][idx]
        par = bundle.ints["parent_id"][idx]
        names = bundle.names
        table = getattr(names, "table", None)
        if table is not None:  # name-id view: test each distinct name once
            flag = names.table_flags(LAYER_NAME_PREFIXES)
            is_layer = flag[names.ids[idx]] if len(flag) else np.zeros(len(idx), bool)
        else:
            is_layer = np.fromiter((_is_layer(names[i], LAYER_NAME_PREFIXES)
                                    for i in idx.tolist()), bool, len(idx))
        lay = np.nonzero(is_layer)[0]
        # ancestor walk, child order and pre-order walk on the device
        # (pm_layer_tree); the layer-name test above stays on the host
        (self.node_parent, o, self.child_off,
         self.walk) = _pipeline.layer_tree(pid, par, is_layer,
                                           bundle.start[idx])
        self.node_event = idx[lay]
        self.node_start = bundle.start[self.node_event]
        self.node_end = bundle.end[self.node_event]
        self.node_name = names.take(self.node_event) if hasattr(names, "take") \
            else [names[i] for i in self.node_event.tolist()]
        self.child_order = o
        self.is_wrapper = np.diff(self.child_off)[1:] > 0
        leaves = self.walk[~self.is_wrapper[self.walk]] if len(lay) else self.walk
        self.leaves = leaves
        self.leaf_start = self.node_start[leaves]
        self.leaf_end = self.node_end[leaves]

    def tree(self) -> tuple[LayerNode, list[LayerNode]]:
        """LayerNode objects (root, leaves in walk order)."""
        nodes = []
        for k in range(len(self.node_event)):
            name = self.node_name[k]
            for prefix in LAYER_NAME_PREFIXES:
                if name.startswith(prefix):
                    name = name[len(prefix):]
                    break
            nodes.append(LayerNode(name=name, start_ts=int(self.node_start[k]),
                                   end_ts=int(self.node_end[k]),
                                   event_id=int(self.node_event[k]),
                                   is_wrapper=bool(self.is_wrapper[k])))
        root = LayerNode(name="<root>", start_ts=0, end_ts=0, is_wrapper=True)
        o, off = self.child_order, self.child_off
        root.children = [nodes[v] for v in o[off[0]:off[1]].tolist()]
        for k, node in enumerate(nodes):
            node.children = [nodes[v] for v in o[off[k + 1]:off[k + 2]].tolist()]
        if root.children:
            root.start_ts = min(c.start_ts for c in root.children)
            root.end_ts = max(c.end_ts for c in root.children)
        return root, [nodes[v] for v in self.leaves.tolist()]
