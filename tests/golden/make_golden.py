"""Generate the golden vectors that pin the oracle and the engine.

Run ONCE in a container where the reference package is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It drives the REFERENCE implementation (peakmem.allocator.AllocatorState,
the same code path replay() uses, allocator.py:155-393) so it can also read
the segment counts and free-pool sizes the reference keeps implicitly.  The
outputs are small JSON files committed next to this script; nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from peakmem.allocator import AllocatorConfig, AllocatorState  # noqa: E402
from peakmem.errors import (DoubleFree, DuplicateHandle,  # noqa: E402
                            MalformedSequence, OutOfMemory, UnknownHandle)
from peakmem import sequencegen as ref_gen  # noqa: E402
from peakmem.orchestration import analyze, build_sequence  # noqa: E402
from peakmem.trace import load_sidecar, parse_trace  # noqa: E402

from oracle import sequencegen as our_gen  # noqa: E402

FIXTURES = Path("/root/reference/pkg/tests/fixtures")


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True,
                                     separators=(",", ":")).encode()).hexdigest()


def run_reference(requests, cfg):
    """replay() (allocator.py:360-393) with segment / pool instrumentation."""
    state = AllocatorState(cfg)
    oom = None
    nseg_peak = 0
    max_pool = 0
    error = None
    for req in requests:
        kind = str(req["kind"]).lower()
        seq_no = req["seq_no"]
        try:
            if kind == "alloc":
                state.allocate(req["block_id"], req["size"], req.get("stream", 0))
            elif kind == "free":
                state.free(req["block_id"])
            else:
                raise MalformedSequence(f"unknown request kind {req['kind']!r}")
        except OutOfMemory:
            oom = seq_no
            nseg_peak = max(nseg_peak, len(state.segments))
            break
        except (UnknownHandle, DoubleFree, DuplicateHandle, MalformedSequence) as exc:
            error = type(exc).__name__
            break
        state.step(seq_no)
        nseg_peak = max(nseg_peak, len(state.segments))
        max_pool = max(max_pool, len(state.free_pool))
    return {
        "peak_reserved": state.peak_reserved,
        "peak_allocated": state.peak_allocated,
        "oom_seq_no": oom,
        "final_reserved": state.reserved_bytes,
        "final_allocated": state.allocated_bytes,
        "n_segments_final": len(state.segments),
        "n_segments_peak": nseg_peak,
        "max_free_blocks": max_pool,
        "timeline_len": len(state.timeline),
        "timeline_sha256": digest([list(t) for t in state.timeline]),
        "error": error,
    }


def corpus_golden(seed, count, config_first):
    rng = random.Random(seed)
    cases = []
    ours = (our_gen.corpus_config_first if config_first else our_gen.corpus)(
        seed, count)
    for i in range(count):
        if config_first:
            params = ref_gen.random_config(rng)
            seq = ref_gen.random_sequence(rng)
        else:
            seq = ref_gen.random_sequence(rng)
            params = ref_gen.random_config(rng)
        assert (seq, params) == ours[i], f"restated generator diverged at {i}"
        cfg = AllocatorConfig(device_capacity=params["capacity"],
                              max_split_size=params["max_split_size"])
        out = run_reference(seq, cfg)
        out["params"] = params
        out["n_requests"] = len(seq)
        out["sequence_sha256"] = digest(seq)
        cases.append(out)
    return {"seed": seed, "count": count, "config_first": config_first,
            "generator": "peakmem.sequencegen (sequencegen.py:15-51)",
            "cases": cases}


def fixture_golden():
    out = {}
    for name in ("tiny_mlp_sgd", "tiny_mlp_adam", "tiny_mlp_sgd_pregrad"):
        root = FIXTURES / name
        bundle = parse_trace(str(root / "trace.json"),
                             sidecar=load_sidecar(str(root / "sidecar.json")))
        seq = build_sequence(analyze(bundle), iterations=2)
        records = seq.replay_records()
        res = run_reference(records, AllocatorConfig())
        # full timeline for these small sequences
        st = AllocatorState(AllocatorConfig())
        for r in records:
            if r["kind"] == "alloc":
                st.allocate(r["block_id"], r["size"], r.get("stream", 0))
            else:
                st.free(r["block_id"])
            st.step(r["seq_no"])
        res["timeline"] = [list(t) for t in st.timeline]
        out[name] = {"records": records, "result": res}
    return out


def main():
    golden = {
        "corpus_seed1000": corpus_golden(1000, 1000, config_first=False),
        "corpus_seed2024": corpus_golden(2024, 300, config_first=False),
        "corpus_seed5eed": corpus_golden(0x5EED, 60, config_first=True),
    }
    for key, val in golden.items():
        (HERE / f"replay_{key}.json").write_text(json.dumps(val, indent=0) + "\n")
    (HERE / "replay_fixture_sequences.json").write_text(
        json.dumps(fixture_golden(), indent=0) + "\n")
    print("wrote", sorted(p.name for p in HERE.glob("replay_*.json")))


if __name__ == "__main__":
    main()
