set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest -x -q -m gpu tests/test_replay_gpu.py tests/test_replay_narrow_gpu.py tests/test_config_goldens.py tests/test_c4_sweep.py tests/test_validate_gpu.py tests/test_capacity.py 2>&1 | tail -4
timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -2
for w in 1 4 6; do
  echo "== pass-1 warps $w"
  PM_PASS1_WARPS=$w timeout 600 python tools/bench_c4.py 2>&1 | tail -1
  PM_PASS1_WARPS=$w timeout 900 python tools/bench_frag.py 2>&1 | tail -1
done
