"""Reference goldens for the allocator configurations the bench and C4 use.

Run ONCE where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_configs.py

Every case is replayed by the REFERENCE (peakmem.allocator.AllocatorState,
driven exactly like replay(), allocator.py:360-393, via make_golden's
run_reference, which also reads segment counts and the free-pool size):

* replay_c4_grid.json -- SURVEY §8d C4: the 69-config grid (max_split_size x
  alignment x segment-size sets) over 4 GPT-2 capture sequences (bs 1/4/8/16,
  2 iterations) and 6 C3 trace prefixes (12k requests of traces 7000-7005);
* replay_multistream.json -- 400 random sequences over 4 streams with all
  eight AllocatorConfig knobs drawn (oracle/sequencegen.py
  multistream_corpus, seed 31337), finite capacities in half of them;
* replay_c3_full.json -- 32 full C3 traces (ids 0, 313, 626, ...; ~1e5
  requests each) at the bench's default config.

Per case: peaks, finals, OOM seq_no, error, segment counts, free-pool high
water, and a timeline digest (c4_cases.timeline_digest: sha256 over int64
rows (seq_no, reserved, allocated)).  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

from peakmem.allocator import AllocatorConfig, AllocatorState  # noqa: E402
from peakmem.errors import (DoubleFree, DuplicateHandle,  # noqa: E402
                            MalformedSequence, OutOfMemory, UnknownHandle)

from c4_cases import c4_grid_params  # noqa: E402
from oracle import c3gen, sequencegen  # noqa: E402

C3_FULL_IDS = list(range(0, 10_000, 313))
C4_C3_IDS = list(range(7000, 7006))
C4_C3_PREFIX = 12_000
MULTISTREAM_SEED, MULTISTREAM_COUNT = 31337, 400


def records_of(reqs) -> list[dict]:
    """Packed records -> the reference's request dicts (seq_no = index)."""
    out = []
    for i, (size, handle, ks) in enumerate(zip(reqs["size"].tolist(),
                                                reqs["handle"].tolist(),
                                                reqs["kind_stream"].tolist())):
        if ks & 3 == 0:
            out.append({"seq_no": i, "kind": "alloc", "block_id": handle,
                        "size": size, "stream": ks >> 2})
        else:
            out.append({"seq_no": i, "kind": "free", "block_id": handle})
    return out


def run(job):
    """One replay through the reference with instrumentation."""
    records, params = job
    state = AllocatorState(AllocatorConfig(**params))
    oom = error = None
    nseg_peak = max_pool = 0
    for req in records:
        kind = str(req["kind"]).lower()
        try:
            if kind == "alloc":
                state.allocate(req["block_id"], req["size"], req.get("stream", 0))
            elif kind == "free":
                state.free(req["block_id"])
            else:
                raise MalformedSequence(kind)
        except OutOfMemory:
            oom = req["seq_no"]
            nseg_peak = max(nseg_peak, len(state.segments))
            break
        except (UnknownHandle, DoubleFree, DuplicateHandle, MalformedSequence) as exc:
            error = type(exc).__name__
            break
        state.step(req["seq_no"])
        nseg_peak = max(nseg_peak, len(state.segments))
        max_pool = max(max_pool, len(state.free_pool))
    rows = np.array(state.timeline, dtype=np.int64).reshape(-1, 3)
    return {
        "peak_reserved": state.peak_reserved,
        "peak_allocated": state.peak_allocated,
        "oom_seq_no": oom,
        "error": error,
        "final_reserved": state.reserved_bytes,
        "final_allocated": state.allocated_bytes,
        "n_segments_final": len(state.segments),
        "n_segments_peak": nseg_peak,
        "max_free_blocks": max_pool,
        "timeline_len": len(rows),
        "timeline_sha256": hashlib.sha256(rows.astype("<i8").tobytes()).hexdigest(),
    }


def seq_digest(reqs) -> str:
    return hashlib.sha256(np.ascontiguousarray(reqs).tobytes()).hexdigest()


def main():
    pool = mp.get_context("fork").Pool()

    # --- C4 grid ----------------------------------------------------------
    z = np.load(HERE / "c2_sequences.npz", allow_pickle=True)
    meta = json.loads(str(z["meta"]))
    traces = []
    for k, m in enumerate(meta):
        if m["iterations"] == 2:
            r = z["reqs"][z["offsets"][k]:z["offsets"][k + 1]]
            traces.append({"name": f"{m['name']}_it2", "source": "c2_sequences.npz",
                           "index": k, "reqs": r})
    for i in C4_C3_IDS:
        traces.append({"name": f"c3_{i}_prefix{C4_C3_PREFIX}", "source": "c3",
                       "index": i, "reqs": c3gen.trace(i)[:C4_C3_PREFIX]})
    grid = c4_grid_params()
    jobs = [(records_of(t["reqs"]), p) for t in traces for p in grid]
    res = pool.map(run, jobs, chunksize=4)
    out = {"configs": grid, "traces": [], "results": []}
    for t in traces:
        out["traces"].append({"name": t["name"], "source": t["source"],
                              "index": t["index"], "n_requests": len(t["reqs"]),
                              "sequence_sha256": seq_digest(t["reqs"])})
    out["results"] = res  # trace-major: result[t * len(grid) + c]
    (HERE / "replay_c4_grid.json").write_text(json.dumps(out, indent=0) + "\n")
    print("c4 grid:", len(res), "replays,",
          len({r["peak_reserved"] for r in res}), "distinct peaks")

    # --- multi-stream, all knobs -------------------------------------------
    cases = sequencegen.multistream_corpus(MULTISTREAM_SEED, MULTISTREAM_COUNT)
    res = pool.map(run, [(seq, cfg) for seq, cfg in cases], chunksize=8)
    for r, (seq, cfg) in zip(res, cases):
        r["params"] = cfg
        r["n_requests"] = len(seq)
        r["sequence_sha256"] = hashlib.sha256(json.dumps(
            seq, sort_keys=True, separators=(",", ":")).encode()).hexdigest()
    (HERE / "replay_multistream.json").write_text(json.dumps(
        {"seed": MULTISTREAM_SEED, "count": MULTISTREAM_COUNT,
         "generator": "oracle/sequencegen.py multistream_corpus",
         "cases": res}, indent=0) + "\n")
    print("multistream:", sum(r["oom_seq_no"] is not None for r in res), "OOM of",
          len(res))

    # --- full C3 traces ----------------------------------------------------
    c3 = [c3gen.trace(i) for i in C3_FULL_IDS]
    res = pool.map(run, [(records_of(r), {}) for r in c3], chunksize=1)
    for r, i, t in zip(res, C3_FULL_IDS, c3):
        r["trace"] = i
        r["n_requests"] = len(t)
        r["sequence_sha256"] = seq_digest(t)
    (HERE / "replay_c3_full.json").write_text(json.dumps(
        {"ids": C3_FULL_IDS, "config": "AllocatorConfig() defaults",
         "generator": "oracle/c3gen.py (numpy PCG64(1_000_003 + i))",
         "cases": res}, indent=0) + "\n")
    print("c3 full:", sum(r["n_requests"] for r in res), "requests")


if __name__ == "__main__":
    main()
