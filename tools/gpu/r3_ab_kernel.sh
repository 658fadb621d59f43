# A/B of two engine builds on C3 (interleaved), an 8-GPU shard and 148 lone traces
A=${1:-base}; B=${2:-exp}
for i in 1 2 3 4; do for v in $A $B; do
  echo -n "$v C3 "; timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
for n in 1250 148; do for v in $A $B; do
  echo -n "$v n=$n "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
