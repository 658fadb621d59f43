python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in 0 6000 4096 3000 2048; do echo "cap $c"; PM_M2_BUCKETS=$c timeout 600 python tools/debug_c5_replay.py 357200 2>&1 | tail -1; done
