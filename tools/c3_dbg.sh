FMG_TRACE=1 timeout 1500 python bench.py --config config3 --steps 2 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c3_dbg.log 2>&1
grep "^{" gpurun_out/c3_dbg.log | tail -1 | cut -c1-200
grep "split\|post" gpurun_out/c3_dbg.log | awk 'NR%2==1' | cut -c1-160 | tail -40
for lib in tools/ab/occ1b.so tools/ab/occ1b_jb.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
done
