"""Summarise an `ncu --set full` capture of the replay kernel into
profiles/replay_ncu_summary.json (read by bench.py for `traffic` and the
issue bound).

    ncu -i prof.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_summary.py raw.csv <events in the profiled launch> "<capture command>" [out.json]
"""

import csv
import json
import sys
from pathlib import Path

STALLS = ["wait", "short_scoreboard", "branch_resolving", "selected", "not_selected",
          "no_instructions", "math_pipe_throttle", "long_scoreboard", "lg_throttle",
          "dispatch_stall", "misc", "mio_throttle", "barrier"]


def num(v):
    return float(v.replace(",", ""))


def main():
    raw, events, capture = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = list(csv.reader(open(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}

    def gbytes(name):
        v, u = get[name]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        return num(v) * scale

    rd, wr = gbytes("dram__bytes_read.sum"), gbytes("dram__bytes_write.sum")
    inst = num(get["smsp__inst_executed.sum"][0])
    samples = {s: num(get[f"smsp__pcsamp_warps_issue_stalled_{s}"][0]) for s in STALLS
               if f"smsp__pcsamp_warps_issue_stalled_{s}" in get}
    tot = sum(samples.values()) or 1.0
    out = {
        "capture": capture,
        "events_in_launch": events,
        "kernel_time_ms": num(get["gpu__time_duration.sum"][0]) / (1e6 if get["gpu__time_duration.sum"][1] == "ns" else 1),
        "registers_per_thread": int(num(get["launch__registers_per_thread"][0])),
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_event": round((rd + wr) / events, 1),
        "warp_instructions_per_event": round(inst / events, 1),
        "smsp_issue_active_pct": round(num(get["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]), 1),
        "warps_active_per_scheduler": round(num(get["smsp__warps_active.avg.per_cycle_active"][0]), 2),
        "thread_inst_per_warp_inst": round(num(get["smsp__thread_inst_executed_per_inst_executed.ratio"][0]), 2)
        if "smsp__thread_inst_executed_per_inst_executed.ratio" in get else None,
        "stall_pct": {s: round(100 * v / tot, 1) for s, v in
                      sorted(samples.items(), key=lambda x: -x[1]) if v / tot > 0.005},
    }
    dest = sys.argv[4] if len(sys.argv) > 4 else "profiles/replay_ncu_summary.json"
    Path(dest).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
