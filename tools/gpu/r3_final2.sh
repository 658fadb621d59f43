# validation after the one-exit change + ncu of the main pass
set -x
TAG=${1:-r3c}
bash tools/gpu/r3_final.sh ${TAG}
bash tools/gpu/r2_ncu.sh ${TAG} > /dev/null 2>&1; echo "ncu rc=$?"
rm -f gpurun_out/${TAG}_replay.ncu-rep
