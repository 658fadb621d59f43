set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench5.log 2> gpurun_out/r2_bench5.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_bench5.err
timeout 1500 python tools/bench_pipeline.py --leaves 6000 60000 357200 > gpurun_out/r2_c5d.jsonl 2> gpurun_out/r2_c5d.err; echo rc=$?; cat gpurun_out/r2_c5d.jsonl; tail -3 gpurun_out/r2_c5d.err
