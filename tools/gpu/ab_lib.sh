# A/B of two engine builds (exp_lib/<a>.so vs exp_lib/<b>.so), interleaved
A=${1:-base}; B=${2:-exp}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2 3; do for v in $A $B; do
  echo -n "$v C3 "; timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
for n in 1 148 1250; do for v in $A $B; do
  echo -n "$v n=$n "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
