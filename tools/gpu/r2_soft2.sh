python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_handoff_gpu.py tests/test_validate_gpu.py -m gpu -q -x 2>&1 | tail -1
timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -1
timeout 600 python tools/debug_c5_replay.py 700000 2>&1 | tail -1
