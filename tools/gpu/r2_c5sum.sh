python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_handoff_gpu.py tests/test_replay_narrow_gpu.py tests/test_validate_gpu.py -m gpu -q -x 2>&1 | tail -1
for c in 0 2048; do echo "cap $c"; PM_M2_BUCKETS=$c timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -1; done
timeout 600 python tools/bench_frag.py 2>&1 | tail -1
