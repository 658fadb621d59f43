"""The reference's sequence-builder cases (pkg/tests/test_orchestration.py:
187-361, TestBuildSequence and TestCloneExtension) restated against this
package: the same conftest iteration layout (tests/pipeline_cases.py
`iteration_records`), the same sidecar and the same expected requests,
timestamps, ids, roles and boundaries.  parse_trace -> analyze ->
build_sequence run through the native reader and the GPU kernels."""

from __future__ import annotations

import json

import pytest

from pipeline_cases import iteration_records

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


@pytest.fixture
def api():
    import paper_2504_03887_b200 as api
    return api


@pytest.fixture
def sidecar(api):
    return api.SidecarConfig(param_sizes=(400,), batch_bytes=(64, 32))


def write(tmp_path, records, name="trace.json"):
    path = tmp_path / name
    path.write_text(json.dumps({"traceEvents": records}))
    return path


@pytest.fixture
def two_iteration_trace(tmp_path):
    return write(tmp_path, iteration_records(0, 0, with_grad_free_at=1025)
                 + iteration_records(1, 1000))


@pytest.fixture
def one_iteration_trace(tmp_path):
    return write(tmp_path, iteration_records(0, 0), "one.json")


@pytest.fixture
def built(api, sidecar):
    def _built(path, iterations=2, side="default"):
        side = sidecar if side == "default" else side
        return api.build_sequence(api.analyze(api.parse_trace(path, sidecar=side)),
                                  iterations=iterations)
    return _built


def by_block(seq, block_id):
    return [r for r in seq.requests if r.block_id == block_id]


class TestBuildSequence:
    def test_request_count_and_seq_nos(self, built, two_iteration_trace):
        assert [r.seq_no for r in built(two_iteration_trace).requests] == list(range(21))

    def test_model_load_first(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        head = seq.requests[0]
        assert (head.block_id, head.size) == ("model:0", 400) and head.virtual_ts < 0
        assert not any(r.kind is api.RequestKind.FREE and r.block_id == "model:0"
                       for r in seq.requests)

    def test_batch_blocks_span_iterations(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        A, F = api.RequestKind.ALLOC, api.RequestKind.FREE
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, "batch:0:1")] == \
            [(A, 0), (F, 900)]
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, "batch:1:0")] == \
            [(A, 1000), (F, 1900)]

    def test_gradient_freed_at_next_zero_grad(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, 3)] == \
            [(api.RequestKind.ALLOC, 250), (api.RequestKind.FREE, 1010)]

    def test_last_iteration_gradient_permanent(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        grad1 = [r for r in seq.requests
                 if seq.phase_tags.get(r.block_id) is api.BlockRole.GRADIENT
                 and r.virtual_ts >= 1000 and r.kind is api.RequestKind.ALLOC]
        assert len(grad1) == 1
        assert not by_block(seq, grad1[0].block_id)[1:]

    def test_optimizer_state_once_and_permanent(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        state = [r for r in seq.requests
                 if seq.phase_tags.get(r.block_id) is api.BlockRole.OPTIMIZER_STATE]
        assert [(r.kind, r.virtual_ts, r.size) for r in state] == \
            [(api.RequestKind.ALLOC, 420, 400)]

    def test_step_span_temporaries_dropped(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        assert 999 not in [r.size for r in seq.requests]
        assert len([r for r in seq.requests
                    if r.kind is api.RequestKind.ALLOC and r.size == 400]) == 4

    def test_intra_op_temporaries_excluded(self, built, two_iteration_trace):
        assert 500 not in [r.size for r in built(two_iteration_trace).requests]

    def test_unclassified_blocks_kept(self, built, two_iteration_trace):
        assert len([r for r in built(two_iteration_trace).requests
                    if r.size == 123]) == 4

    def test_boundaries(self, built, two_iteration_trace):
        assert built(two_iteration_trace).iteration_boundaries == [0, 1000, 1900]

    def test_allocs_precede_frees(self, api, built, two_iteration_trace):
        seen = set()
        for r in built(two_iteration_trace).requests:
            if r.kind is api.RequestKind.ALLOC:
                assert r.block_id not in seen
                seen.add(r.block_id)
            else:
                assert r.block_id in seen

    def test_free_before_alloc_at_same_ts(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        by_ts: dict = {}
        for r in seq.requests:
            by_ts.setdefault(r.virtual_ts, []).append(r)
        alloc_at = {r.block_id: r.virtual_ts for r in seq.requests
                    if r.kind is api.RequestKind.ALLOC}
        for group in by_ts.values():
            ranks = [1 if r.kind is api.RequestKind.ALLOC
                     else (0 if alloc_at[r.block_id] < r.virtual_ts else 2)
                     for r in group]
            assert ranks == sorted(ranks)

    def test_deterministic(self, built, two_iteration_trace):
        assert built(two_iteration_trace).to_json_dict() == \
            built(two_iteration_trace).to_json_dict()

    def test_replayable(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace)
        res = api.replay(seq.replay_records(),
                         api.AllocatorConfig(max_split_size=1 << 62))
        assert res.oom_seq_no is None and res.peak_reserved > 0

    def test_single_iteration_request(self, api, built, two_iteration_trace):
        seq = built(two_iteration_trace, iterations=1)
        assert seq.iteration_boundaries == [0, 1000]
        assert not [r for r in seq.requests
                    if r.virtual_ts >= 1000 and r.kind is api.RequestKind.ALLOC]
        assert len([r for r in seq.requests
                    if str(r.block_id).startswith("batch:")]) == 4

    def test_zero_iterations_rejected(self, api, built, two_iteration_trace):
        with pytest.raises(api.NoIterations):
            built(two_iteration_trace, iterations=0)

    def test_missing_sidecar_rejected(self, api, built, two_iteration_trace):
        with pytest.raises(api.MissingBatchBytes):
            built(two_iteration_trace, side=None)


class TestCloneExtension:
    def test_cloned_blocks_fresh_ids_and_shift(self, api, built, one_iteration_trace):
        seq = built(one_iteration_trace)
        A, F = api.RequestKind.ALLOC, api.RequestKind.FREE
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, 0)] == [(A, 70), (F, 230)]
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, "clone1:0")] == \
            [(A, 970), (F, 1130)]

    def test_clone_creates_no_optimizer_state(self, api, built, one_iteration_trace):
        seq = built(one_iteration_trace)
        assert [b for b, role in seq.phase_tags.items()
                if role is api.BlockRole.OPTIMIZER_STATE] == [4]

    def test_original_gradient_freed_at_cloned_zero_grad(self, api, built,
                                                         one_iteration_trace):
        seq = built(one_iteration_trace)
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, 3)] == \
            [(api.RequestKind.ALLOC, 250), (api.RequestKind.FREE, 910)]

    def test_cloned_gradient_permanent(self, api, built, one_iteration_trace):
        seq = built(one_iteration_trace)
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, "clone1:3")] == \
            [(api.RequestKind.ALLOC, 1150)]

    def test_batch_blocks_cover_cloned_iteration(self, api, built, one_iteration_trace):
        seq = built(one_iteration_trace)
        assert [(r.kind, r.virtual_ts) for r in by_block(seq, "batch:1:0")] == \
            [(api.RequestKind.ALLOC, 900), (api.RequestKind.FREE, 1800)]

    def test_boundaries_extend_past_trace(self, built, one_iteration_trace):
        assert built(one_iteration_trace).iteration_boundaries == [0, 900, 1800]

    def test_alloc_multisets_match(self, api, built, one_iteration_trace):
        seq = built(one_iteration_trace)
        b = seq.iteration_boundaries
        first = sorted(r.size for r in seq.requests
                       if r.kind is api.RequestKind.ALLOC
                       and b[0] <= r.virtual_ts < b[1]
                       and seq.phase_tags[r.block_id] is not api.BlockRole.OPTIMIZER_STATE)
        second = sorted(r.size for r in seq.requests
                        if r.kind is api.RequestKind.ALLOC and b[1] <= r.virtual_ts < b[2])
        assert first == second
