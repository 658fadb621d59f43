python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest -x -q -m gpu tests/test_handoff_gpu.py tests/test_replay_gpu.py 2>&1 | tail -15
