set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for v in 0 1; do
  echo "== PM_LONG_1B=$v"
  PM_LONG_1B=$v timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -2
  PM_LONG_1B=$v timeout 600 python tools/debug_c5_replay.py 60000 2>&1 | tail -1
done
timeout 900 python -m pytest -x -q -m gpu tests/test_pipeline_gpu.py tests/test_handoff_gpu.py tests/test_replay_narrow_gpu.py 2>&1 | tail -2
