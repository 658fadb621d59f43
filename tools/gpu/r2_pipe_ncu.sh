# ncu --set full of the batched pipeline's top kernels at 10^7 events (C5):
# the layer tree's CTA-per-node passes, the warp-cooperative link, the
# breakdown (a first capture with DeviceRadixSortOnesweep in the filter took
# six CUB sort passes, profiles/r02_pipeline_ncu_sort.json).  Raw pages are
# summarised by tools/ncu_pipe_summary.py into profiles/.
set -x
TAG=${1:-r2p}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none \
  -k regex:'k_preorder_big|k_link_fwd|k_breakdown|k_subtree_big' \
  -c 5 -o gpurun_out/${TAG}_pipe \
  python tools/profile_batch.py 357200 > gpurun_out/${TAG}_pipe_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_pipe_ncu.log
ncu -i gpurun_out/${TAG}_pipe.ncu-rep --page raw --csv > gpurun_out/${TAG}_pipe_raw.csv
ls -la gpurun_out/ | grep ${TAG}
