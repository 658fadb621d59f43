"""Drop the B200 engine into a running reference `peakmem` pipeline.

The reference estimator binds `replay`, `analyze` and `build_sequence` into
its module namespace at import (pkg/src/peakmem/estimator.py:9,12-17) and
calls them at estimator.py:146 and :152; the CLI calls
`peakmem.allocator.replay` (cli.py:188).  `install()` rebinds those names to
GPU-backed wrappers that take and return the reference's own types
(records / AllocatorConfig / TraceBundle in, SimulationResult /
AnalyzedTrace-compatible objects out) and raise the reference's own
exception classes, so `PeakMemoryEstimator.estimate(bundle)` and
`peakmem replay` run on the GPU unchanged.  `uninstall()` restores them.

    import peakmem
    from paper_2504_03887_b200 import plugin
    plugin.install()                      # replay on the GPU
    plugin.install(pipeline=True)         # + analyze / build_sequence
"""

from __future__ import annotations

import functools
import importlib
import sys

from . import errors as _our_errors
from .allocator import replay as _gpu_replay

_saved: dict = {}


def _translate(fn, ref_errors):
    """Re-raise engine exceptions as the reference's classes of the same
    name (errors.py:11-82)."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except _our_errors.PeakMemError as exc:
            cls = getattr(ref_errors, type(exc).__name__, None)
            if cls is None:
                raise
            raise cls(str(exc)) from exc
    return wrapper


def _ref_replay(ref_allocator, ref_errors):
    def replay(requests, cfg=None, validate=False):
        out = _gpu_replay(requests, cfg, validate)
        return ref_allocator.SimulationResult(
            peak_reserved=out.peak_reserved, peak_allocated=out.peak_allocated,
            timeline=out.timeline, oom_seq_no=out.oom_seq_no,
            final_reserved=out.final_reserved,
            final_allocated=out.final_allocated)
    return _translate(replay, ref_errors)


def _ref_bundle(bundle):
    """Reference TraceBundle -> the engine's columnar bundle."""
    from .trace import parse_records, SidecarConfig
    recs = bundle.to_json_dict()["traceEvents"]
    meta = bundle.metadata
    side = None if meta is None else SidecarConfig(
        param_sizes=tuple(meta.param_sizes), batch_bytes=tuple(meta.batch_bytes),
        optimizer_name=meta.optimizer_name, device_capacity=meta.device_capacity,
        initial_memory=meta.initial_memory)
    return parse_records(recs, bundle.source_path, side)


def install(pipeline: bool = False, module: str = "peakmem") -> None:
    """Rebind the reference's replay (and optionally analyze /
    build_sequence) to the GPU engine."""
    ref = importlib.import_module(module)
    ref_est = importlib.import_module(f"{module}.estimator")
    ref_alloc = importlib.import_module(f"{module}.allocator")
    ref_errors = importlib.import_module(f"{module}.errors")
    gpu_replay = _ref_replay(ref_alloc, ref_errors)
    targets = [(ref_est, "replay", gpu_replay), (ref_alloc, "replay", gpu_replay),
               (ref, "replay", gpu_replay)]
    if pipeline:
        from . import orchestration as ours
        ref_orch = importlib.import_module(f"{module}.orchestration")
        ref_analysis = importlib.import_module(f"{module}.analysis")
        ref_build = _original(ref_orch, "build_sequence")

        def analyze(bundle):
            return ours.analyze(_ref_bundle(bundle))

        def build_sequence(analyzed, iterations=2):
            if not isinstance(analyzed, ours.AnalyzedTrace):
                # an AnalyzedTrace the reference built itself (e.g. before
                # install()): its own enums and objects, its own function
                return ref_build(analyzed, iterations)
            seq = ours.build_sequence(analyzed, iterations)
            kinds = {"alloc": ref_orch.RequestKind.ALLOC,
                     "free": ref_orch.RequestKind.FREE}
            reqs = [ref_orch.MemoryRequest(
                seq_no=r.seq_no, kind=kinds[r.kind.value], block_id=r.block_id,
                size=r.size, virtual_ts=r.virtual_ts, stream=r.stream)
                for r in seq.requests]
            tags = {k: ref_analysis.BlockRole(v.value)
                    for k, v in seq.phase_tags.items()}
            return ref_orch.RequestSequence(
                requests=reqs, iteration_boundaries=seq.iteration_boundaries,
                phase_tags=tags)

        # every alias of the pair moves together (estimator.py:12-17 binds
        # them at import, __init__.py:71 re-exports them), so the reference's
        # own build_sequence never sees the engine's AnalyzedTrace
        gpu_analyze = _translate(analyze, ref_errors)
        gpu_build = _translate(build_sequence, ref_errors)
        for mod in (ref_est, ref_orch, ref):
            targets += [(mod, "analyze", gpu_analyze),
                        (mod, "build_sequence", gpu_build)]
    cli = sys.modules.get(f"{module}.cli")
    if cli is not None:  # cli.py:24 binds replay at import (used at :188)
        targets.append((cli, "replay", gpu_replay))
    for mod, name, fn in targets:
        key = (mod.__name__, name)
        _saved.setdefault(key, (mod, getattr(mod, name)))
        setattr(mod, name, fn)


def _original(mod, name):
    """The reference's own function, even if install() already ran."""
    saved = _saved.get((mod.__name__, name))
    return saved[1] if saved else getattr(mod, name)


def uninstall() -> None:
    for (_, name), (mod, fn) in list(_saved.items()):
        setattr(mod, name, fn)
    _saved.clear()
