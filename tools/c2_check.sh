timeout 900 python -m pytest tests -m gpu -x -q -k "z1 or bidirectional or scale_golden_config2 or inexact" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200; done
