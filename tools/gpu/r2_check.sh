set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r2_gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench1.log 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench1.log; tail -5 gpurun_out/r2_bench1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_ref1.log 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r2_ref1.log
