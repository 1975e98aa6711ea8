timeout 900 python -m pytest tests -m gpu -x -q -k "z1 or bidirectional or scale_golden_config2 or inexact" 2>&1 | tail -2
for lib in paper_1811_06127_b200/libfmgpu.so tools/ab/jumpb.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
  FMG_LIB_PATH=$lib timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130
done
