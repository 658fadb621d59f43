set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for sp in 0 1; do
  echo "== PM_SPREAD=$sp"
  for n in 64 500 1250 1776 3500; do
    PM_SPREAD=$sp timeout 300 python tools/prof_replay.py --traces $n --launches 4 2>&1 | tail -1
  done
  PM_SPREAD=$sp timeout 300 python tools/bench_c2.py --ref-sample 0 2>&1 | tail -1 | cut -c1-260
done
timeout 900 python -m pytest -x -q -m gpu tests/test_replay_gpu.py tests/test_captures.py tests/test_c4_sweep.py 2>&1 | tail -2
