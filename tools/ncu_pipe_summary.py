"""Summarise an `ncu --set full` capture of the batched pipeline's kernels
(tools/gpu/r2_pipe_ncu.sh) into one row per launch: duration, DRAM bytes,
achieved DRAM bandwidth, SM / issue activity, warps per scheduler, the top
stall reasons.

    ncu -i pipe.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_pipe_summary.py raw.csv [out.json]
"""

import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "branch_resolving",
          "barrier", "membar", "lg_throttle", "mio_throttle", "math_pipe_throttle",
          "no_instructions", "selected", "not_selected", "dispatch_stall", "misc",
          "drain", "sleeping", "imc_miss", "tex_throttle"]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}

        def q(name):
            v, u = get[name]
            return num(v) * SCALE.get(u, 1.0)

        t = q("gpu__time_duration.sum")
        dram = q("dram__bytes_read.sum") + q("dram__bytes_write.sum")
        samples = {s: num(get[f"smsp__pcsamp_warps_issue_stalled_{s}"][0])
                   for s in STALLS if f"smsp__pcsamp_warps_issue_stalled_{s}" in get}
        tot = sum(samples.values()) or 1.0
        top = sorted(samples.items(), key=lambda kv: -kv[1])[:4]
        name = get["Kernel Name"][0]
        out.append({
            "kernel": name[:90],
            "grid": get.get("Grid Size", ("", ""))[0],
            "block": get.get("Block Size", ("", ""))[0],
            "us": round(t * 1e6, 2),
            "dram_mb": round(dram / 1e6, 3),
            "dram_gbs": round(dram / t / 1e9, 1) if t else None,
            "sm_busy_pct": num(get.get("sm__throughput.avg.pct_of_peak_sustained_elapsed",
                                       ("nan", ""))[0]),
            "issue_active_pct": num(get.get("smsp__issue_active.avg.pct_of_peak_sustained_active",
                                            ("nan", ""))[0]),
            "warps_per_scheduler": num(get.get("smsp__warps_active.avg.per_cycle_active",
                                               ("nan", ""))[0]),
            "stalls_pct": {k: round(100 * v / tot, 1) for k, v in top},
        })
    text = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
