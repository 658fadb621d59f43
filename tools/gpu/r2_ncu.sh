# ncu capture of the replay main pass: one full wave (3552 C3 traces), source
# counters for the per-line instruction profile, plus the raw page.
set -x
TAG=${1:-r2a}
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:replay_narrow_kernel -s 1 -c 1 -o gpurun_out/${TAG}_replay \
  python tools/prof_replay.py --traces 3552 --launches 2 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log
ncu -i gpurun_out/${TAG}_replay.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv
ncu -i gpurun_out/${TAG}_replay.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null || \
ncu -i gpurun_out/${TAG}_replay.ncu-rep --page source --csv > gpurun_out/${TAG}_sass.csv
ls -la gpurun_out/
