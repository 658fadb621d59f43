set -x
TAG=${1:-r2g}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest -x -q -m gpu tests/test_replay_gpu.py tests/test_replay_narrow_gpu.py tests/test_config_goldens.py tests/test_handoff_gpu.py tests/test_validate_gpu.py tests/test_batch_edges_gpu.py 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python tools/prof_replay.py --traces 10000 --launches 3 2>&1 | tail -1; done
bash tools/gpu/r2_ncu.sh ${TAG} > /dev/null 2>&1; echo "ncu rc=$?"
