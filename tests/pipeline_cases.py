"""Pipeline parity inputs: generated traces and the reference's hand-laid
iteration layout (pkg/tests/conftest.py:50-89), restated as data."""

from __future__ import annotations

import hashlib
import json

from oracle import tracegen


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True,
                                     separators=(",", ":")).encode()).hexdigest()

CASES = [
    {"name": "gen_s1", "seed": 1},
    {"name": "gen_s2_sgd", "seed": 2, "kw": {"optimizer": "sgd"}},
    {"name": "gen_s3_pregrad", "seed": 3, "kw": {"zero_grad": "pre-backward"}},
    {"name": "gen_s4_one_iter", "seed": 4, "kw": {"iterations": 1}},
    {"name": "gen_s5_big", "seed": 5, "kw": {"layers": 40, "leaves": 4}},
    {"name": "gen_s6_two_iter", "seed": 6, "kw": {"iterations": 2}},
    {"name": "gen_s7_wide", "seed": 7, "kw": {"layers": 2, "leaves": 12}},
    {"name": "gen_s8_sgd_one", "seed": 8, "kw": {"optimizer": "sgd", "iterations": 1}},
    {"name": "gen_s9_int_ts", "seed": 9, "kw": {"jitter_ts": False}},
    {"name": "gen_s10", "seed": 10, "kw": {"layers": 12, "leaves": 2, "iterations": 4}},
    {"name": "gen_s11", "seed": 11},
    {"name": "gen_s12_pregrad_one", "seed": 12,
     "kw": {"zero_grad": "pre-backward", "iterations": 1}},
    {"name": "gen_s13", "seed": 13, "kw": {"layers": 24, "leaves": 3}},
    {"name": "gen_s14", "seed": 14, "kw": {"layers": 3, "leaves": 1}},
    {"name": "gen_s15_int_sgd", "seed": 15, "kw": {"jitter_ts": False, "optimizer": "sgd"}},
    {"name": "gen_s16", "seed": 16, "kw": {"layers": 60, "leaves": 4, "iterations": 2}},
    {"name": "conftest_two_iter", "conftest": True},
]


def ev(cat, name, ts, dur=None, **args):
    rec = {"ph": "i" if cat == "cpu_instant_event" else "X",
           "cat": cat, "name": name, "ts": ts, "args": args}
    if dur is not None:
        rec["dur"] = dur
    return rec


def instant(ts, addr, nbytes):
    return ev("cpu_instant_event", "[memory]", ts, Addr=addr, Bytes=nbytes)


def iteration_records(k, base, with_grad_free_at=None, with_span_blocks=True):
    """One iteration of the reference conftest's layout at `base`
    (pkg/tests/conftest.py:50-89, restated): ProfilerStep [0, 900),
    zero-grad at +10, a Linear forward at +60 with a retained 1000 B
    activation and a 500 B intra-op temporary, an unowned 123 B block at
    +150, backward at +200 with a 400 B gradient, an optimizer step
    [+400, +500) with an optional surviving 400 B state block and two
    span-local temporaries."""
    pid, seq = 10 + k, 100 + k
    recs = [
        ev("user_annotation", f"ProfilerStep#{k}", base, 900),
        ev("user_annotation", "Optimizer.zero_grad#SGD.zero_grad", base + 10, 20),
        ev("python_function", "nn.Module: Linear_0", base + 50, 100,
           **{"Python id": pid}),
        ev("cpu_op", "aten::linear", base + 60, 50, **{"Sequence number": seq}),
        instant(base + 70, 0x1000 + k, 1000),
        instant(base + 72, 0x2000 + k, 500),
        instant(base + 80, 0x2000 + k, -500),
        instant(base + 150, 0x7000 + k, 123),
        ev("cpu_op", "autograd::engine::evaluate_function: AddmmBackward0",
           base + 200, 100, **{"Sequence number": seq}),
        instant(base + 230, 0x1000 + k, -1000),
        instant(base + 250, 0x3000 + k, 400),
        ev("user_annotation", "Optimizer.step#SGD.step", base + 400, 100),
        instant(base + 600, 0x7000 + k, -123),
    ]
    if with_span_blocks:
        recs += [instant(base + 420, 0x4000 + k, 400),
                 instant(base + 430, 0x5000 + k, 999),
                 instant(base + 440, 0x5000 + k, -999),
                 instant(base + 435, 0x6000 + k, 400),
                 instant(base + 450, 0x6000 + k, -400)]
    if with_grad_free_at is not None:
        recs.append(instant(with_grad_free_at, 0x3000 + k, -400))
    return recs


def _conftest_records():
    """Two iterations of the reference conftest layout at base 0 and 1000,
    the first with a gradient free at +1010 (test_orchestration.py)."""
    recs = (iteration_records(0, 0, with_grad_free_at=1010)
            + iteration_records(1, 1000))
    side = {"param_sizes": [400], "batch_bytes": [128, 64], "optimizer": "sgd",
            "device_capacity_bytes": 0, "initial_memory_bytes": 0}
    return recs, side


def case_records(case):
    if case.get("conftest"):
        return _conftest_records()
    return tracegen.generate(case["seed"], **case.get("kw", {}))


def views(api, bundle) -> dict:
    """Everything the reference exposes, reduced to comparable JSON; `api`
    is either package (same names)."""
    a = api.analyze(bundle)
    walk = [n for n in a.layer_tree.walk()]
    leaf_index = {n: i for i, n in enumerate(
        [n for n in walk if n is not a.layer_tree and not n.is_wrapper])}

    def layer(n):
        d = {"name": n.name, "start": n.start_ts, "end": n.end_ts,
             "wrapper": n.is_wrapper, "children": [layer(c) for c in n.children]}
        p = a.profiles.get(n)
        if p is not None:
            d["fwd"] = [a.operator_roots.index(op) for op in p.forward_ops]
            d["bwd"] = [a.operator_roots.index(op) for op in p.backward_ops]
            d["ret"] = [b.block_id for b in p.retained_blocks]
            d["tmp"] = [b.block_id for b in p.temporary_blocks]
        return d

    events = [[e.category.value, e.start_ts, e.duration, e.name]
              for e in bundle.events]
    roots = [[op.name, op.start_ts, op.end_ts, sorted(op.sequence_numbers)]
             for op in a.operator_roots]
    markers = [[m.kind.value, m.start_ts, m.end_ts, m.iteration_index]
               for m in a.markers]
    blocks = [[b.block_id, b.addr, b.size, b.alloc_time, b.free_time,
               b.role.value] for b in a.blocks]
    out = {
        "n_events": len(bundle.events),
        "events_sha256": digest(events),
        "layers_sha256": digest(layer(a.layer_tree)),
        "n_roots": len(roots), "roots_sha256": digest(roots),
        "markers": markers,
        "n_blocks": len(blocks), "blocks_sha256": digest(blocks),
        "bundle_json_sha256": digest(bundle.to_json_dict()),
    }
    for it in (1, 2, 3):
        a2 = api.analyze(bundle)
        try:
            seq = api.build_sequence(a2, iterations=it)
        except Exception as exc:  # noqa: BLE001
            out[f"seq{it}"] = {"error": type(exc).__name__}
            continue
        after = [[b.block_id, b.free_time, b.role.value] for b in a2.blocks]
        out[f"seq{it}"] = {
            "n": len(seq.requests),
            "req_sha256": digest([[r.kind.value, r.block_id, r.size, r.virtual_ts]
                                  for r in seq.requests]),
            "sha256": digest(seq.to_json_dict()),
            "boundaries": seq.iteration_boundaries,
            "blocks_after_sha256": digest(after),
        }
    for name, kw in (("default", {}), ("cap", {"device_capacity": 64 << 20}),
                     ("split", {"max_split_size": 32 << 20, "iterations": 3})):
        try:
            out[f"report_{name}"] = api.PeakMemoryEstimator(**kw).estimate(
                bundle).canonical_json()
        except Exception as exc:  # noqa: BLE001
            out[f"report_{name}"] = {"error": type(exc).__name__}
    return out


