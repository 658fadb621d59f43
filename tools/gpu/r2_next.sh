set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest -x -q -m gpu tests/test_host_pack_gpu.py tests/test_batch_edges_gpu.py tests/test_replay_gpu.py tests/test_capi.py 2>&1 | tail -4
PM_REPLAY_WARPS=1 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2_racecheck_w1.log 2>&1; echo "racecheck w1 rc=$?"; tail -3 gpurun_out/r2_racecheck_w1.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench4.log 2> gpurun_out/r2_bench4.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2_bench4.log; tail -3 gpurun_out/r2_bench4.err
bash tools/gpu/r2_flags.sh 2>&1 | grep -v "^+"
