set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests5.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/r2_gputests5.log; grep -E "FAILED|Error" gpurun_out/r2_gputests5.log | head
timeout 1500 python tools/bench_pipeline.py --leaves 6000 60000 357200 > gpurun_out/r2_c5c.jsonl 2> gpurun_out/r2_c5c.err; echo rc=$?; cat gpurun_out/r2_c5c.jsonl; tail -3 gpurun_out/r2_c5c.err
