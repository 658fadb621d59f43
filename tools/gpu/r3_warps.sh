# C3 at pinned main-pass widths (PM_REPLAY_WARPS) and the 2-GPU shard size
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2; do for w in 24 28 20; do
  echo -n "warps=$w C3 "; PM_REPLAY_WARPS=$w timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -1
done; done
for n in 5000 2500 1250; do echo -n "n=$n "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1; done
