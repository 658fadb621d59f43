set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests2.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/r2_gputests2.log
timeout 900 python tools/profile_batch.py 357200 > gpurun_out/r2_profile_batch2.txt 2>&1; head -30 gpurun_out/r2_profile_batch2.txt
timeout 1500 python tools/bench_pipeline.py --sweep 64 --leaves 6000 60000 357200 > gpurun_out/r2_c5b.jsonl 2> gpurun_out/r2_c5b.err
echo rc=$?; cat gpurun_out/r2_c5b.jsonl; tail -3 gpurun_out/r2_c5b.err
