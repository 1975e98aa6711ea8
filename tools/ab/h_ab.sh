for lib in tools/ab/h10.so tools/ab/h11.so tools/ab/h12.so tools/ab/h13.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 4 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
  FMG_LIB_PATH=$lib FMG_BIDIR_MIN_N=0 timeout 600 python -m pytest tests -m gpu -x -q -k "bidirectional and split" 2>&1 | tail -1
done
