# ncu source counters of the one-warp main-pass CTA on 148 C3 traces (one per SM)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_narrow_kernel -s 1 -c 1 \
  -o gpurun_out/r3_w1_148 python tools/prof_replay.py --traces 148 --launches 2 > gpurun_out/r3_w1_148.log 2>&1; echo rc=$?
ncu -i gpurun_out/r3_w1_148.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r3_w1_148_cs.csv 2>/dev/null; echo src rc=$?
rm -f gpurun_out/r3_w1_148.ncu-rep
