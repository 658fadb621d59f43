set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_replay_narrow_gpu.py tests/test_handoff_gpu.py tests/test_c4_sweep.py -m gpu -q -x 2>&1 | tail -2
for n in 148 1776 1777 2000 2368 2369 2600 2960 2961 3552 10000; do
  echo -n "n=$n: "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1
done
for n in 2000 2600; do for w in 16 20 24; do
  echo -n "n=$n W=$w: "; PM_REPLAY_WARPS=$w timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1
done; done
