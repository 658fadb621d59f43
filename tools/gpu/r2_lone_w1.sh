# ncu of the one-warp main-pass CTA on a lone C3 trace and on 148 traces
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for n in 1 148; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_narrow_kernel -s 1 -c 1 \
  -o gpurun_out/r2_w1_${n} python tools/prof_replay.py --traces $n --launches 2 > gpurun_out/r2_w1_${n}.log 2>&1; echo rc=$?
ncu -i gpurun_out/r2_w1_${n}.ncu-rep --page raw --csv > gpurun_out/r2_w1_${n}_raw.csv
tail -1 gpurun_out/r2_w1_${n}.log
done
