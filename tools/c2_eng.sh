for e in split sync dfs; do
  echo "=== $e"
  FMG_BIDIR_ENGINE=$e FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 5 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>&1 | grep "^\[fmg\]" | tail -2 | cut -c1-200
  FMG_BIDIR_ENGINE=$e timeout 600 python bench.py --config config2 --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-130
done
