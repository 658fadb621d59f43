# C2 end to end on the box: capture the 64 GPT-2 traces, then reference vs
# engine on the same files (tools/bench_c2_e2e.py), with a cProfile of the
# batched engine path.
set -x
TAG=${1:-r2k}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python tools/bench_c2_e2e.py --capture --jobs 4 --profile > gpurun_out/${TAG}_c2e2e.json 2> gpurun_out/${TAG}_c2e2e.err
echo rc=$?; cat gpurun_out/${TAG}_c2e2e.json
