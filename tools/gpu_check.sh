set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_gputest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_bench_fast.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/r02_bench_fast.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exact > gpurun_out/r02_bench_exact.log 2>&1; echo "bench exact rc=$?"
tail -2 gpurun_out/r02_bench_exact.log
