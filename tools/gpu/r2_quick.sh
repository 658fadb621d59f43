# quick iteration: build, replay parity tests, C3 10^4-trace timing
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest -x -q -m gpu tests/test_replay_gpu.py tests/test_replay_narrow_gpu.py tests/test_config_goldens.py tests/test_c4_sweep.py ${EXTRA_TESTS} 2>&1 | tail -4
timeout 600 python tools/prof_replay.py --traces 10000 --launches 4 2>&1 | tail -3
