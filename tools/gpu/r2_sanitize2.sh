# compute-sanitizer over the main-pass widths: default (one-warp / 12-warp
# CTAs for these small batches) and PM_SPREAD=0 (24-warp CTAs)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2s_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/r2s_racecheck.log
PM_SPREAD=0 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2s_racecheck_packed.log 2>&1; echo "racecheck packed rc=$?"; tail -4 gpurun_out/r2s_racecheck_packed.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_replay.py > gpurun_out/r2s_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2s_memcheck.log
PM_SPREAD=0 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_replay.py > gpurun_out/r2s_memcheck_packed.log 2>&1; echo "memcheck packed rc=$?"; tail -3 gpurun_out/r2s_memcheck_packed.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_replay.py > gpurun_out/r2s_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/r2s_synccheck.log
