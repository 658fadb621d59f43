set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest -q -m gpu tests/test_pipeline_gpu.py -k "1e6" 2>&1 | tail -2
timeout 1500 python tools/bench_pipeline.py --leaves 36000 357200 --file > gpurun_out/r2_c5.jsonl 2> gpurun_out/r2_c5.err
echo rc=$?; cat gpurun_out/r2_c5.jsonl; tail -3 gpurun_out/r2_c5.err
