set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2_racecheck2.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/r2_racecheck2.log
PM_REPLAY_WARPS=1 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2_racecheck_1warp.log 2>&1; echo "racecheck 1-warp rc=$?"; tail -4 gpurun_out/r2_racecheck_1warp.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_replay.py > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2_memcheck.log
timeout 1200 compute-sanitizer --tool memcheck python -m pytest -x -q -m gpu tests/test_batch_gpu.py tests/test_layer_tree_gpu.py > gpurun_out/r2_memcheck_pipe.log 2>&1; echo "memcheck pipeline rc=$?"; tail -4 gpurun_out/r2_memcheck_pipe.log
