# config-3-style z=1 pass (14M seeds, 3.1 Gbp): split (default) vs level-synchronous form, with the engine trace
mkdir -p gpurun_out
for e in split sync; do
  echo "=== engine $e"
  FMG_BIDIR_ENGINE=$e FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 4 2>&1 | grep -v "pre-engine" | tail -12
done
