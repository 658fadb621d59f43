"""The reference's own unit cases for analysis and linking
(pkg/tests/test_analysis.py:45-248, pkg/tests/test_linking.py:39-190),
restated against this package's API: same inputs, same expected values.
Markers are host code (CPU tests); the layer tree, operator roots,
grouping and the three link steps run on the GPU (pm_layer_tree / pm_link /
pm_link_roots)."""

from __future__ import annotations

import itertools

import pytest

from paper_2504_03887_b200.analysis import (AnnotationMarker, BlockRole,
                                            LayerNode, MarkerKind, MemoryBlock,
                                            OperatorNode, build_layer_tree,
                                            build_operator_roots,
                                            extract_markers,
                                            group_memory_events)
from paper_2504_03887_b200.errors import CyclicParentLink, NoIterationMarkers
from paper_2504_03887_b200.linking import (attach_backward_ops, attach_blocks,
                                           link, link_layers_to_ops)
from paper_2504_03887_b200.trace import EventCategory, TraceEvent

_ids = itertools.count()
gpu = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def fn(name, ts, dur, python_id, parent_id=None):
    return TraceEvent(next(_ids), EventCategory.PYTHON_FUNCTION, name, ts, dur,
                      python_id=python_id, parent_id=parent_id)


def op(name, ts, dur, seq=None):
    return TraceEvent(next(_ids), EventCategory.CPU_OP, name, ts, dur,
                      sequence_number=seq)


def ann(name, ts, dur):
    return TraceEvent(next(_ids), EventCategory.USER_ANNOTATION, name, ts, dur)


def mem(ts, addr, nbytes):
    return TraceEvent(next(_ids), EventCategory.CPU_INSTANT_EVENT, "[memory]", ts,
                      0, addr=addr, nbytes=nbytes)


# ---- layer tree (test_analysis.py:45-104), GPU (pm_layer_tree) ----------------

@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_root_with_two_children():
    tree = build_layer_tree([fn("nn.Module: Sequential_0", 0, 100, 1),
                             fn("nn.Module: Linear_0", 10, 20, 2, 1),
                             fn("nn.Module: ReLU_0", 40, 10, 3, 1)])
    assert len(tree.children) == 1
    seq = tree.children[0]
    assert seq.name == "Sequential_0"
    assert [c.name for c in seq.children] == ["Linear_0", "ReLU_0"]


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_non_layer_frame_collapsed():
    tree = build_layer_tree([
        fn("nn.Module: Block_0", 0, 100, 1),
        fn("torch/nn/functional.py(1843): relu", 5, 90, 2, 1),
        fn("nn.Module: Linear_0", 10, 20, 3, 2)])
    assert tree.children[0].name == "Block_0"
    assert [c.name for c in tree.children[0].children] == ["Linear_0"]


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_orphan_attaches_to_root():
    tree = build_layer_tree([fn("nn.Module: Linear_0", 0, 10, 1, 999)])
    assert [c.name for c in tree.children] == ["Linear_0"]


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_wrapper_flag():
    tree = build_layer_tree([fn("nn.Module: Sequential_0", 0, 100, 1),
                             fn("nn.Module: Linear_0", 10, 20, 2, 1)])
    assert tree.children[0].is_wrapper
    assert not tree.children[0].children[0].is_wrapper


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_cycle_detected():
    with pytest.raises(CyclicParentLink):
        build_layer_tree([fn("nn.Module: A_0", 0, 10, 1, 2),
                          fn("plain", 0, 10, 2, 1)])


def test_tree_rejects_wrong_category():
    with pytest.raises(ValueError):
        build_layer_tree([op("aten::add", 0, 1)])


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_tree_children_sorted_by_time():
    tree = build_layer_tree([fn("nn.Module: B_0", 50, 10, 2),
                             fn("nn.Module: A_0", 0, 10, 1)])
    assert [c.name for c in tree.children] == ["A_0", "B_0"]


# ---- markers (test_analysis.py:156-200) ---------------------------------------

def test_markers_two_iterations():
    markers = extract_markers([ann("ProfilerStep#0", 0, 100),
                               ann("Optimizer.zero_grad#SGD.zero_grad", 10, 5),
                               ann("Optimizer.step#SGD.step", 60, 20),
                               ann("ProfilerStep#1", 100, 90)])
    steps = [m for m in markers if m.kind is MarkerKind.PROFILER_STEP]
    assert [m.iteration_index for m in steps] == [0, 1]
    assert next(m for m in markers if m.kind is MarkerKind.ZERO_GRAD).iteration_index == 0
    assert next(m for m in markers
                if m.kind is MarkerKind.OPTIMIZER_STEP).iteration_index == 0


def test_markers_second_iteration():
    markers = extract_markers([ann("ProfilerStep#0", 0, 100),
                               ann("ProfilerStep#1", 100, 90),
                               ann("Optimizer.zero_grad#SGD.zero_grad", 110, 5)])
    assert next(m for m in markers if m.kind is MarkerKind.ZERO_GRAD).iteration_index == 1


def test_markers_no_zero_grad():
    markers = extract_markers([ann("ProfilerStep#0", 0, 100)])
    assert all(m.kind is not MarkerKind.ZERO_GRAD for m in markers)


def test_markers_no_steps_is_error():
    with pytest.raises(NoIterationMarkers):
        extract_markers([ann("Optimizer.step#SGD.step", 0, 10)])


def test_markers_unrelated_ignored():
    assert len(extract_markers([ann("ProfilerStep#0", 0, 100),
                                ann("my_custom_region", 5, 10)])) == 1


def test_markers_are_values():
    assert AnnotationMarker(MarkerKind.PROFILER_STEP, 0, 10, 0) == \
        AnnotationMarker(MarkerKind.PROFILER_STEP, 0, 10, 0)


# ---- operator roots (test_analysis.py:107-153), GPU ----------------------------

@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestOperatorRoots:
    def test_containment(self):
        roots = build_operator_roots([op("A", 0, 10), op("B", 2, 3), op("C", 20, 10)])
        assert [r.name for r in roots] == ["A", "C"]

    def test_nested_seq_absorbed(self):
        roots = build_operator_roots([op("A", 0, 10), op("B", 2, 3, seq=7)])
        assert roots[0].sequence_numbers == {7}

    def test_own_and_absorbed_merge(self):
        roots = build_operator_roots([op("A", 0, 10, seq=3), op("B", 2, 3, seq=7)])
        assert roots[0].sequence_numbers == {3, 7}

    def test_closed_open_boundary(self):
        roots = build_operator_roots([op("A", 0, 10), op("B", 10, 5)])
        assert [r.name for r in roots] == ["A", "B"]

    def test_deeply_nested(self):
        roots = build_operator_roots([op("A", 0, 100), op("B", 10, 50, seq=1),
                                      op("C", 20, 10, seq=2)])
        assert len(roots) == 1 and roots[0].sequence_numbers == {1, 2}

    def test_identical_intervals_first_wins(self):
        roots = build_operator_roots([op("A", 0, 10), op("B", 0, 10, seq=4)])
        assert [r.name for r in roots] == ["A"]
        assert roots[0].sequence_numbers == {4}

    def test_pairwise_non_nested(self):
        roots = build_operator_roots([op("A", 0, 10), op("B", 3, 2),
                                      op("C", 10, 10), op("D", 25, 5)])
        for a in roots:
            for b in roots:
                if a is not b:
                    assert not (b.start_ts <= a.start_ts and a.end_ts <= b.end_ts)


# ---- grouping (test_analysis.py:203-248), GPU ----------------------------------

@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestGrouping:
    def test_alloc_free_pair(self):
        b, = group_memory_events([mem(1, 0x10, 512), mem(5, 0x10, -512)])
        assert (b.addr, b.size, b.alloc_time, b.free_time) == (0x10, 512, 1, 5)
        assert not b.permanent

    def test_unmatched_alloc_permanent(self):
        assert group_memory_events([mem(1, 0x10, 512)])[0].permanent

    def test_address_reuse(self):
        blocks = group_memory_events([mem(1, 0x10, 512), mem(2, 0x10, -512),
                                      mem(3, 0x10, 1024), mem(9, 0x10, -1024)])
        assert [(b.alloc_time, b.free_time) for b in blocks] == [(1, 2), (3, 9)]

    def test_orphan_free_dropped(self):
        blocks = group_memory_events([mem(1, 0x10, -512), mem(2, 0x20, 256)])
        assert len(blocks) == 1 and blocks[0].addr == 0x20

    def test_double_alloc_closes_then_opens(self):
        first, second = group_memory_events([mem(1, 0x10, 512), mem(4, 0x10, 1024)])
        assert first.free_time == 4 and second.permanent

    def test_block_count_equals_alloc_count(self):
        events = [mem(1, 1, 100), mem(2, 2, 200), mem(3, 1, -100),
                  mem(4, 1, 300), mem(5, 3, -999)]
        assert len(group_memory_events(events)) == 3

    def test_ids_follow_alloc_order(self):
        blocks = group_memory_events([mem(5, 1, 100), mem(1, 2, 200)])
        assert [b.block_id for b in blocks] == [0, 1]
        assert [b.alloc_time for b in blocks] == [1, 5]

    def test_size_from_alloc_event(self):
        assert group_memory_events([mem(1, 1, 512), mem(2, 1, -768)])[0].size == 512

    def test_role_starts_unclassified(self):
        b = group_memory_events([mem(1, 1, 512)])[0]
        assert isinstance(b, MemoryBlock) and b.role.value == "unclassified"


# ---- linking (test_linking.py:39-190), GPU -------------------------------------

def layer(name, start, end, children=(), wrapper=False):
    return LayerNode(name=name, start_ts=start, end_ts=end,
                     children=list(children), is_wrapper=wrapper)


def tree_of(*layers):
    return LayerNode(name="<root>", start_ts=0, end_ts=10_000,
                     children=list(layers), is_wrapper=True)


def node(name, start, end, seqs=()):
    return OperatorNode(name=name, start_ts=start, end_ts=end,
                        sequence_numbers=set(seqs))


def block(block_id, alloc, free=None, size=512):
    return MemoryBlock(block_id=block_id, addr=block_id, size=size,
                       alloc_time=alloc, free_time=free)


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestLinkLayersToOps:
    def test_layer_owns_contained_ops(self):
        lin = layer("Linear_0", 0, 100)
        a, b = node("A", 5, 10), node("B", 50, 60)
        assert link_layers_to_ops(tree_of(lin), [a, b])[lin].forward_ops == [a, b]

    def test_innermost_wins(self):
        inner = layer("Linear_0", 10, 20)
        outer = layer("Custom_0", 0, 100, children=[inner])
        o = node("O", 12, 15)
        p = link_layers_to_ops(tree_of(outer), [o])
        assert p[inner].forward_ops == [o] and p[outer].forward_ops == []

    def test_wrapper_excluded(self):
        inner = layer("Linear_0", 10, 20)
        wrapper = layer("Sequential_0", 0, 100, children=[inner], wrapper=True)
        o = node("O", 12, 15)
        p = link_layers_to_ops(tree_of(wrapper), [o])
        assert wrapper not in p and p[inner].forward_ops == [o]

    def test_outside_unowned(self):
        lin = layer("Linear_0", 0, 100)
        assert link_layers_to_ops(tree_of(lin), [node("O", 200, 210)])[lin].forward_ops == []

    def test_partial_overlap_not_owned(self):
        lin = layer("Linear_0", 0, 100)
        assert link_layers_to_ops(tree_of(lin), [node("O", 90, 110)])[lin].forward_ops == []


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestAttachBackwardOps:
    def _run(self, lin, ops):
        p = link_layers_to_ops(tree_of(lin), ops)
        attach_backward_ops(p, ops)
        return p[lin].backward_ops

    def test_single_seq(self):
        fwd, bwd = node("aten::linear", 5, 10, {3}), node("AddmmBackward0", 500, 520, {3})
        assert self._run(layer("Linear_0", 0, 100), [fwd, bwd]) == [bwd]

    def test_union_over_seqs(self):
        f1, f2 = node("f1", 5, 10, {3}), node("f2", 20, 30, {4})
        b1, b2 = node("b1", 500, 510, {3}), node("b2", 520, 530, {4})
        assert self._run(layer("Custom_0", 0, 100), [f1, f2, b1, b2]) == [b1, b2]

    def test_no_seq_no_backward(self):
        assert self._run(layer("ReLU_0", 0, 100), [node("aten::relu", 5, 10)]) == []

    def test_own_forward_not_reattached(self):
        assert self._run(layer("Linear_0", 0, 100), [node("aten::linear", 5, 10, {3})]) == []

    def test_dedup_by_identity(self):
        f1, shared = node("f1", 5, 10, {3, 4}), node("b", 500, 510, {3, 4})
        assert self._run(layer("Custom_0", 0, 100), [f1, shared]) == [shared]


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
class TestAttachBlocks:
    def _one(self, alloc, free):
        lin = layer("Linear_0", 0, 100)
        p = link_layers_to_ops(tree_of(lin), [node("O", 10, 20)])
        b = block(0, alloc=alloc, free=free)
        attach_blocks(p, [b])
        return p[lin], b

    def test_temporary_inside_one_op(self):
        prof, b = self._one(12, 18)
        assert prof.temporary_blocks == [b] and b.role is BlockRole.TEMPORARY

    def test_retained_outlives_op(self):
        prof, b = self._one(12, 500)
        assert prof.retained_blocks == [b] and b.role is BlockRole.RETAINED

    def test_permanent_is_retained(self):
        prof, b = self._one(12, None)
        assert prof.retained_blocks == [b]

    def test_before_any_op_unclassified(self):
        prof, b = self._one(5, None)
        assert b.role is BlockRole.UNCLASSIFIED and prof.retained_blocks == []

    def test_free_at_op_end_is_retained(self):
        _, b = self._one(12, 20)
        assert b.role is BlockRole.RETAINED

    def test_partition_property(self):
        lin1, lin2 = layer("Linear_0", 0, 100), layer("Linear_1", 200, 300)
        p = link_layers_to_ops(tree_of(lin1, lin2),
                               [node("O1", 10, 20), node("O2", 210, 260)])
        blocks = [block(0, 12, 15), block(1, 12, 500), block(2, 220),
                  block(3, 150), block(4, 999)]
        attach_blocks(p, blocks)
        placed = (p[lin1].retained_blocks + p[lin1].temporary_blocks
                  + p[lin2].retained_blocks + p[lin2].temporary_blocks)
        unclassified = [b for b in blocks if b.role is BlockRole.UNCLASSIFIED]
        assert len(placed) + len(unclassified) == len(blocks)
        assert {id(b) for b in placed} | {id(b) for b in unclassified} == \
            {id(b) for b in blocks}

    def test_backward_owner_only_after_attach(self):
        """Owners are the profile's owned ops at call time: a block born in
        a backward op is attached only once backward ops are attached."""
        lin = layer("Linear_0", 0, 100)
        ops = [node("f", 5, 10, {3}), node("b", 500, 520, {3})]
        p = link_layers_to_ops(tree_of(lin), ops)
        b = block(0, alloc=505)
        attach_blocks(p, [b])
        assert b.role is BlockRole.UNCLASSIFIED
        p = link_layers_to_ops(tree_of(lin), ops)
        attach_backward_ops(p, ops)
        b = block(0, alloc=505)
        attach_blocks(p, [b])
        assert b.role is BlockRole.RETAINED


@pytest.mark.gpu
@pytest.mark.usefixtures("require_gpu")
def test_backward_retained_gradient_candidates():
    lin = layer("Linear_0", 0, 100)
    fwd = node("aten::linear", 5, 10, {3})
    bwd = node("AddmmBackward0", 500, 520, {3})
    p = link(tree_of(lin), [fwd, bwd], [block(0, 6, 900), block(1, 505, None),
                                        block(2, 507, 510)])
    assert [b.block_id for b in p[lin].backward_retained_blocks()] == [1]
