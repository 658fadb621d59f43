set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python tools/profile_batch.py 357200 > gpurun_out/r2_profile_batch.txt 2>&1; tail -50 gpurun_out/r2_profile_batch.txt
timeout 1500 python tools/bench_pipeline.py --leaves 6000 60000 357200 > gpurun_out/r2_c5.jsonl 2> gpurun_out/r2_c5.err
echo rc=$?; cat gpurun_out/r2_c5.jsonl; tail -3 gpurun_out/r2_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv python tools/profile_batch.py 357200 > /dev/null 2>&1; echo ncu rc=$?
