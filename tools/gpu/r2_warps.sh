set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for w in 20 24 28 32; do
  echo "== warps $w"
  PM_REPLAY_WARPS=$w timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -2
done
