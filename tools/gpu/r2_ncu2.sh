# round-2 evidence: ncu --set full of the main replay kernel (one wave of C3)
# + the bench launch list (gpu__time_duration per launch)
set -x
TAG=${1:-r2b}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
bash tools/gpu/r2_ncu.sh $TAG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launches rc=$?"
