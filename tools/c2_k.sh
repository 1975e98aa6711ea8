for v in "FMG_X=0" "FMG_LUT_K=12" "FMG_LUT_K=11" "FMG_LIB_PATH=tools/ab/nojump.so" "FMG_LIB_PATH=tools/ab/nojump.so FMG_LUT_K=11"; do
  echo "=== $v"
  env $v FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 5 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>&1 | grep "split" | tail -1 | cut -c1-170
  env $v timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130
done
