set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python tools/bench_c4.py --check 2>&1 | tail -1
timeout 900 python -m pytest -x -q -m gpu tests/test_c4_sweep.py tests/test_handoff_gpu.py tests/test_replay_gpu.py tests/test_replay_narrow_gpu.py tests/test_config_goldens.py tests/test_capacity.py tests/test_validate_gpu.py tests/test_captures.py 2>&1 | tail -3
for b in 0 1; do
  echo "== PM_BESIDE=$b"
  PM_BESIDE=$b timeout 600 python tools/bench_c4.py 2>&1 | tail -1
  PM_BESIDE=$b timeout 600 python tools/bench_frag.py 2>&1 | tail -1
  PM_BESIDE=$b timeout 300 python tools/prof_replay.py --traces 3500 --launches 3 2>&1 | tail -1
  PM_BESIDE=$b timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -1
done
