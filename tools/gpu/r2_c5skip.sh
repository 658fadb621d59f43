python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -2
PM_LONG_SKIP=0 timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -2
