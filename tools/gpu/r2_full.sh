# full GPU suite, the bench line (with other configs), the reference arm,
# racecheck / memcheck on the sanitizer batches
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests3.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/r2_gputests3.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench3.log 2> gpurun_out/r2_bench3.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench3.log; tail -3 gpurun_out/r2_bench3.err
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_replay.py > gpurun_out/r2_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/r2_racecheck.log
