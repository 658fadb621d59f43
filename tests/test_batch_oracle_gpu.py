"""GPU: the batched pipeline against the CPU oracle (oracle/pipeline.py,
itself pinned to the reference's goldens) on batches of randomly
parameterised generated traces.  Every generated trace starts near the same
timestamp with the same python ids, sequence numbers and addresses, so the
batch's isolation by rebasing is exercised on every join: a leak between
traces would change some trace's requests."""

from __future__ import annotations

import json
import random

import numpy as np
import pytest

import paper_2504_03887_b200 as api
from oracle import pipeline as op
from oracle import tracegen
from paper_2504_03887_b200.batch import build_sequences
from paper_2504_03887_b200.orchestration import _block_id

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("require_gpu")]


def _cases(n, seed):
    rng = random.Random(seed)
    out = []
    for k in range(n):
        kw = {"iterations": rng.choice([1, 2, 3, 4]), "layers": rng.choice([2, 3, 6, 12, 24]),
              "leaves": rng.choice([1, 2, 3, 5]), "optimizer": rng.choice(["adam", "sgd"]),
              "zero_grad": rng.choice(["start", "pre-backward"]),
              "jitter_ts": rng.random() < 0.7}
        out.append((seed * 1000 + k, kw))
    return out


def _bundle(recs, side, tmp_path, name):
    p = tmp_path / f"{name}.json"
    p.write_text(json.dumps({"traceEvents": recs}))
    sc = api.SidecarConfig(param_sizes=tuple(side["param_sizes"]),
                           batch_bytes=tuple(side["batch_bytes"]),
                           optimizer_name=side["optimizer"])
    return api.parse_trace(p, sidecar=sc)


@pytest.mark.parametrize("it", [1, 2, 3])
def test_random_batches_vs_oracle(tmp_path, it):
    cases = _cases(24, 40 + it)
    recs_sides = [tracegen.generate(s, **kw) for s, kw in cases]
    bundles = [_bundle(r, sd, tmp_path, f"t{k}") for k, (r, sd) in enumerate(recs_sides)]
    batch = build_sequences(bundles, iterations=it, views=True)
    v = {f: (t.cpu().numpy() if hasattr(t, "cpu") else t) for f, t in batch.views.items()}
    for k, (recs, side) in enumerate(recs_sides):
        try:
            want = op.build_sequence(op.normalize(recs), side, it)
        except Exception as exc:  # noqa: BLE001 -- the class must match
            assert type(batch.errors[k]).__name__ == type(exc).__name__, (k, batch.errors[k])
            continue
        assert batch.errors[k] is None, (k, batch.errors[k])
        a, b = int(batch.req_off[k]), int(batch.req_off[k + 1])
        kinds = ("alloc", "free")
        got = [(kinds[int(kd)], _block_id(int(tg), int(x), int(y)), int(sz), int(vt))
               for kd, tg, x, y, sz, vt in zip(v["kind"][a:b], v["tag"][a:b], v["a"][a:b],
                                               v["b"][a:b], v["size"][a:b], v["vts"][a:b])]
        assert got == want, (k, cases[k])
        # the packed replay records of the trace are its own, handles dense
        pk = batch.packed(k)
        assert len(pk) == b - a
        assert int(pk["handle"].max()) < len(pk)
