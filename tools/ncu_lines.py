"""Aggregate an ncu SASS source page (CSV) by CUDA source line.

    ncu -i prof.ncu-rep --page source --csv > sass.csv
    python tools/ncu_lines.py sass.csv lib.so <kernel-substring> [top]

Maps each SASS instruction (by offset from the function start) to the
source line nvdisasm reports for the same cubin (-lineinfo builds).
"""

import collections
import csv
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def line_map(so: str, kernel_sub: str):
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(so).resolve())], cwd=tmp, check=True,
                   capture_output=True)
    out = {}
    for cubin in tmp.glob("*.cubin"):
        txt = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)],
                             capture_output=True, text=True).stdout
        func = None
        cur = None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                func = m.group(1)
                continue
            m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
            if m:
                cur = (Path(m.group(1)).name, int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and func and kernel_sub in func:
                out.setdefault(func, {})[int(m.group(1), 16)] = cur
    return out


def main():
    sass_csv, so, ksub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    data = rows[2:]
    ia = hdr.index("Address")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    maps = line_map(so, ksub)
    if not maps:
        sys.exit("kernel not found in cubin")
    fmap = max(maps.values(), key=len)
    base = int(data[0][ia], 16)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        off = int(r[ia], 16) - base
        key = fmap.get(off, ("?", 0))
        agg[key][0] += int(r[isamp] or 0)
        agg[key][1] += int(r[iex] or 0)
    ts = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {ts}  total warp-instructions {te}")
    for (f, ln), (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100*s/ts:6.2f}% samp {100*e/te:6.2f}% inst  {f}:{ln}")


if __name__ == "__main__":
    main()
