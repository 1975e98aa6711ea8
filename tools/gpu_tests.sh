(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>&1 | grep -v "^\[fmg\] \(bidir\|inexact post\)" | tail -1 | cut -c1-130; done
FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
