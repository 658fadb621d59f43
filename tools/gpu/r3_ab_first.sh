# A/B: first-wave trace assignment warp-major by position (exp, -DPM_FIRST_SPREAD)
# vs the atomic counter (base); C3 sweep, an 8-GPU-sized shard, C4
A=${1:-base}; B=${2:-exp}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2 3; do for v in $A $B; do
  echo -n "$v C3 "; timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
for n in 1250 3552; do for v in $A $B; do
  echo -n "$v n=$n "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
for v in $A $B $A $B; do
  echo "$v C4 "; timeout 300 python tools/bench_c4.py --reps 5 --check --lib exp_lib/$v.so 2>&1 | tail -3
done
