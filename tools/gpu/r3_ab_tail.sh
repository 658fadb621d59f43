# A/B: C4's packed one-wave batch with the long/short first-wave split (default)
# vs the atomic counter (PM_TAIL_CTAS=0); then the replay GPU tests
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2 3; do
  echo "split C4"; timeout 300 python tools/bench_c4.py --reps 5 --check 2>&1 | tail -1
  echo "counter C4"; PM_TAIL_CTAS=0 timeout 300 python tools/bench_c4.py --reps 5 --check 2>&1 | tail -1
done
for v in 1 0; do echo -n "tail=$v n=3552 "; PM_TAIL_CTAS=$v timeout 300 python tools/prof_replay.py --traces 3552 --launches 3 2>&1 | tail -1; done
echo -n "C3 "; timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "replay or batch or narrow or c4 or c2 or handoff or capacity" > gpurun_out/r3_tail_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_tail_tests.log
