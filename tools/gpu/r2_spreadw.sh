# small batches (spread one CTA per SM): main-pass instantiation with fewer
# warps (more registers) vs the default 24
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for n in 148 600 1250 1776; do
  for w in 24 12 16 20 1; do
    [ "$w" = 1 ] && [ "$n" -gt 148 ] && continue
    echo -n "n=$n W=$w: "; PM_REPLAY_WARPS=$w timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1
  done
done
