set -x
for cfg in "PM_REPLAY_WIDE=1" "PM_REPLAY_WARPS=12" "PM_REPLAY_WARPS=16" "PM_REPLAY_WARPS=20"; do
  env $cfg timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -2
done
