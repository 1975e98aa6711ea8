timeout 900 python -m pytest tests -m gpu -x -q -k "validation or inexact_random or small_cases or exact_edge" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130; done
