# A/B: under-a-wave batches start by position (exp = the tree's build) vs HEAD~ (base)
A=${1:-base}; B=${2:-exp}
for n in 1250 2500 600 148 1250 2500; do for v in $A $B; do
  echo -n "$v n=$n "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done; done
for v in $A $B; do
  echo -n "$v C3 "; timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 --lib exp_lib/$v.so 2>&1 | tail -1
done
timeout 900 python -m pytest tests -m gpu -q -x -k "replay or batch or narrow or c4 or c2 or shard or bench" > gpurun_out/r3_pos_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pos_tests.log
