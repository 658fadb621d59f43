"""Goldens from real training-step captures.

Captures come from tools/capture_models.py (torch CPU profiler; not
committed raw).  Run where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_captures.py

Writes tests/golden/captures_golden.json (reference views + reports for the
ResNet-18 bs32 and GPT-2 bs8 traces, whose gzipped traces are committed
under tests/golden/traces/) and tests/golden/c2_sequences.npz (the packed
GPT-2 request sequences of batch sizes 1/4/8/16 at 2 and 10 iterations,
with the reference's replay results incl. segment counts).
"""

from __future__ import annotations

import gzip
import json
import logging
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
sys.path.insert(0, str(HERE))
logging.disable(logging.WARNING)

import peakmem  # noqa: E402
from peakmem.allocator import AllocatorConfig  # noqa: E402
from peakmem.orchestration import analyze, build_sequence  # noqa: E402
from peakmem.trace import load_sidecar, parse_trace  # noqa: E402

from make_golden import run_reference  # noqa: E402
from paper_2504_03887_b200.allocator import pack_trace  # noqa: E402
from pipeline_cases import views  # noqa: E402

CAPS = REPO / "data" / "captures"
COMMITTED = ("resnet18_bs32_224", "gpt2_bs8_s128")
C2 = ("gpt2_bs1_s128", "gpt2_bs4_s128", "gpt2_bs8_s128", "gpt2_bs16_s128")


def main():
    gold = {}
    for name in COMMITTED:
        src = CAPS / name
        with open(src / "trace.json", "rb") as f, gzip.open(
                HERE / "traces" / f"{name}.trace.json.gz", "wb", 9) as g:
            shutil.copyfileobj(f, g)
        shutil.copy(src / "sidecar.json", HERE / "traces" / f"{name}.sidecar.json")
        bundle = parse_trace(str(src / "trace.json"),
                             sidecar=load_sidecar(str(src / "sidecar.json")))
        gold[name] = views(peakmem, bundle)
        print(name, gold[name]["n_events"], "events")
    (HERE / "captures_golden.json").write_text(json.dumps(gold, indent=0) + "\n")
    packed, offs, meta = [], [0], []
    for name in C2:
        src = CAPS / name
        bundle = parse_trace(str(src / "trace.json"),
                             sidecar=load_sidecar(str(src / "sidecar.json")))
        for it in (2, 10):
            recs = build_sequence(analyze(bundle), iterations=it).replay_records()
            res = run_reference(recs, AllocatorConfig())
            p = pack_trace(recs)
            packed.append(p.reqs)
            offs.append(offs[-1] + len(p.reqs))
            meta.append({"name": name, "iterations": it, **res})
            print(name, it, len(recs), res["peak_reserved"], res["n_segments_peak"])
    np.savez_compressed(HERE / "c2_sequences.npz", reqs=np.concatenate(packed),
                        offsets=np.array(offs, dtype=np.int64),
                        meta=np.array(json.dumps(meta)))


if __name__ == "__main__":
    main()
