set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log
timeout 900 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-600
timeout 1500 python bench.py --config config3 --steps 2 --warmup 3 --no-hbm-extra > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-600
