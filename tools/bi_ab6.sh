for lib in paper_1811_06127_b200/libfmgpu.so tools/ab/jb6.so tools/ab/b6.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
done
