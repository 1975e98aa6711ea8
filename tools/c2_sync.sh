timeout 900 python -m pytest tests -m gpu -x -q -k "z1 or bidirectional or scale_golden_config2 or inexact or config2" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130; done
