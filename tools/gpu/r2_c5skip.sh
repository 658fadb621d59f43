# C5's lone trace: default routing (main pass -> passes 1 / 1b -> 2 with checkpoints)
# vs PM_LONG_SKIP=1 (straight to narrow pass 2, the round-1 rule)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -2
PM_LONG_SKIP=1 timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -2
