set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_narrow_kernel -s 1 -c 1 -o gpurun_out/r2_lone python tools/prof_replay.py --traces 148 --launches 2 > gpurun_out/r2_lone.log 2>&1; echo rc=$?
ncu -i gpurun_out/r2_lone.ncu-rep --page raw --csv > gpurun_out/r2_lone_raw.csv
