set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest -q -m gpu tests/test_captures.py 2>&1 | tail -2
timeout 900 python tools/bench_c2.py --ref-sample 8 > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err
echo rc=$?; cat gpurun_out/r2_c2.json; tail -3 gpurun_out/r2_c2.err
