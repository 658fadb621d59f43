# adaptive main-pass width for small batches: GPU suite + sizes sweep
set -x
TAG=${1:-r2w}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log
for n in 1 16 148 149 600 1250 1776 1777 2500 3552 10000; do
  echo -n "n=$n: "; timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1
  echo -n "n=$n packed: "; PM_SPREAD=0 timeout 300 python tools/prof_replay.py --traces $n --launches 3 2>&1 | tail -1
done
timeout 600 python tools/bench_c4.py 2>&1 | tail -1
timeout 600 python tools/bench_frag.py 2>&1 | tail -1
