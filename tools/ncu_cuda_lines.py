"""Per-CUDA-line stall samples / instructions from an ncu report's
"cuda,sass" source view (needs -lineinfo; uses the cubin inside the report).

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > cs.csv
    python tools/ncu_cuda_lines.py cs.csv <events> [top]
"""
import collections
import csv
import sys


def main():
    path, events = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    fname, hdr = None, None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0].isdigit():
            continue
        # columns: Line No, Source, Address, Source(sass), metrics...
        line, src = int(r[0]), r[1]
        try:
            samp = float(r[4] or 0)
            inst = float(r[7] or 0)
        except ValueError:
            continue
        a = agg[(fname, line)]
        a[0] += samp
        a[1] += inst
        a[2] = src
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"samples {ts:.0f}  warp-instructions/event {ti / events:.1f}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * s / ts:5.2f}% {i / events:6.2f}/ev  {f}:{ln}  {src.strip()[:70]}")


if __name__ == "__main__":
    main()
