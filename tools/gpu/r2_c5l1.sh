set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for nb in 0 4096 3072 2048; do
  echo "== pass-2 buckets $nb"
  PM_PASS2_BUCKETS=$nb timeout 600 python tools/debug_c5_replay.py 300000 2>&1 | tail -2
done
