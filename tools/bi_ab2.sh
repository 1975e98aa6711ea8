# A/B of k_inexact_bi variants on config 3 (1M reads = 14M seeds); FMG_LIB_PATH per variant
for lib in paper_1811_06127_b200/libfmgpu.so tools/ab/u0.so tools/ab/minb6.so tools/ab/old.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
done
