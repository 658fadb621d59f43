# Main-kernel width sweep on the C3 workload (10^4 traces); one process per
# setting because the launch configuration is fixed per process.
set -x
for cfg in ${SWEEP:-"PM_REPLAY_WIDE=1" "PM_REPLAY_WARPS=12" "PM_REPLAY_WARPS=16" "PM_REPLAY_WARPS=20" "PM_REPLAY_WARPS=24"}; do
  env $cfg timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -2
done
