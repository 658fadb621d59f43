"""Device layer tree (pm_layer_tree) against the CPU
oracle's restatement of analysis.py:113-182 on randomised python_function
forests: non-layer frames to collapse, orphans, duplicate python ids (first
wins), start-time ties (event id breaks them) and parent cycles."""

from __future__ import annotations

import random

import pytest

from oracle import pipeline as op
from paper_2504_03887_b200.errors import CyclicParentLink
from paper_2504_03887_b200.trace import EventCategory, TraceEvent

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def forest(rng: random.Random, n: int, cyc: bool):
    ids = list(range(1, n + 1))
    rng.shuffle(ids)
    evs = []
    for k in range(n):
        pid = ids[k]
        if rng.random() < 0.05:
            pid = rng.choice(ids)  # duplicate id
        if rng.random() < 0.03:
            pid = None
        r = rng.random()
        if r < 0.15:
            par = None
        elif r < 0.2:
            par = 10_000 + k       # orphan: parent never seen
        else:
            par = ids[rng.randrange(0, max(1, k))] if k else None
        if cyc and k < 3:
            par = ids[(k + 1) % 3]
        layer = rng.random() < 0.6
        name = (f"nn.Module: L{k}" if layer else
                rng.choice(["torch/nn/modules/module.py(1500): _call_impl",
                            "helper.py(3): f", "<built-in method x>"]))
        start = rng.randrange(0, 50)
        evs.append((k, name, start, rng.randrange(0, 20), pid, par))
    order = list(range(n))
    rng.shuffle(order)  # list order != event id order
    return [evs[i] for i in order]


def shape(node, key):
    return (key(node), [shape(c, key) for c in node])


def test_layer_tree_matches_oracle_on_random_forests():
    from paper_2504_03887_b200.analysis import build_layer_tree
    rng = random.Random(4)
    cyclic_seen = 0
    for case in range(300):
        cyc = rng.random() < 0.1
        evs = forest(rng, rng.randrange(1, 120), cyc)
        te = [TraceEvent(k, EventCategory.PYTHON_FUNCTION, name, s, d,
                         python_id=pid, parent_id=par)
              for (k, name, s, d, pid, par) in evs]
        od = [{"cat": "python_function", "name": name, "start": s, "end": s + d,
               "pid": pid, "parent": par, "id": k}
              for (k, name, s, d, pid, par) in evs]
        try:
            want_root, want_leaves = op.layer_tree(od)
        except ValueError:
            cyclic_seen += 1
            with pytest.raises(CyclicParentLink):
                build_layer_tree(te)
            continue
        got = build_layer_tree(te)

        def g(n):
            return (n.name, n.start_ts, n.end_ts, n.is_wrapper,
                    [g(c) for c in n.children])

        def w(n):
            return (n["name"], n["start"], n["end"], n["wrapper"],
                    [w(c) for c in n["children"]])
        assert g(got) == w(want_root), case
        leaves = [n for n in got.walk() if n is not got and not n.is_wrapper]
        assert [(n.name, n.start_ts) for n in leaves] == \
            [(n["name"], n["start"]) for n in want_leaves], case
    assert cyclic_seen > 5
