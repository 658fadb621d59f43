# C4: long traces per long CTA in the first-wave split (PM_TAIL_PER_CTA)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2; do for k in 24 22 20 18; do
  echo -n "per_cta=$k "; PM_TAIL_PER_CTA=$k timeout 300 python tools/bench_c4.py --reps 5 --check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['device_ms'], d['retry_passes'][:3], d['oracle_equal'])"
done; done
