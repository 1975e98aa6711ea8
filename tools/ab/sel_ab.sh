timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for lib in paper_1811_06127_b200/libfmgpu.so tools/ab/oldsel.so; do
  echo "=== lib=$lib"
  FMG_LIB_PATH=$lib timeout 600 python tools/exact_latency.py 1000000 1,10000 2>&1 | grep "m 13\|m 32"
  FMG_LIB_PATH=$lib FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 4 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
  for c in config0 config2; do FMG_LIB_PATH=$lib timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value']/1e6)"; done
done
