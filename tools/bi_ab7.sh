timeout 900 python -m pytest tests -m gpu -x -q -k "bidirectional or z1 or repeated" 2>&1 | tail -2
for lib in paper_1811_06127_b200/libfmgpu.so tools/ab/jumpb.so; do
 for ow in 1 0; do
  echo "=== lib=$lib oneword=$ow"
  FMG_BI_ONEWORD=$ow FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
 done
done
