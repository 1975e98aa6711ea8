timeout 900 python -m pytest tests -m gpu -x -q -k "z1 or bidirectional or config2 or inexact or small_cases" 2>&1 | tail -2
FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 5 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>&1 | grep "^\[fmg\]" | tail -1 | cut -c1-200
for i in 1 2; do timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130; done
