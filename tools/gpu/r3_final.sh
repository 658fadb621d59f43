# session-3 validation: smoke, GPU suite, bench line + reference arm, bench
# launch list, C5 routing, pipeline-kernel ncu
set -x
TAG=${1:-r3}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/${TAG}_gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/${TAG}_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-other-configs \
  > /dev/null 2>&1; echo "launches rc=$?"


