# config 2 A/B: level-synchronous z1 (default for L2-resident) vs bidirectional split vs DFS
for v in "FMG_X=0" "FMG_INEXACT_DFS=1" "FMG_INEXACT_DFS=1 FMG_INEXACT_BIDIR=0"; do
  echo "=== $v"
  env $v FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 3 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>&1 | grep -v "^{" | tail -4
  env $v timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
done
