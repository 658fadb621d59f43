set -x
python tools/stats_replay.py 3552 > gpurun_out/r2_stats_c3.log 2>&1
python tools/stats_replay.py 10000 > gpurun_out/r2_stats_c3b.log 2>&1
cat gpurun_out/r2_stats_c3.log gpurun_out/r2_stats_c3b.log | grep -v "^ptxas\|^nvcc"
