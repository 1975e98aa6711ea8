# config 2 engine trace: default vs bidir off
for v in "" "FMG_INEXACT_BIDIR=0"; do
  echo "=== $v"
  env $v FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 3 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>&1 | grep -v "^{" | tail -30
  env $v timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300
done
