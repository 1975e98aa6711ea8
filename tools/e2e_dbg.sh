timeout 900 python -m pytest tests -m gpu -x -q -k "bidirectional or z1 or repeated or inexact or config2 or validation" 2>&1 | tail -2
for e in sync split; do
  echo "== engine $e"
  FMG_BIDIR_ENGINE=$e timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, d['e2e']['value']/1e6)"
done
FMG_TRACE=1 timeout 1500 python bench.py --config config3 --steps 2 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c3_dbg2.log 2>&1
grep "^{" gpurun_out/c3_dbg2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value']/1e6, d['e2e']['value']/1e6)"
grep "split" gpurun_out/c3_dbg2.log | sed 's/.*B sort + merge \([0-9.]*\) ms.*/\1/' | sort -n | tail -5 | tr '\n' ' '
