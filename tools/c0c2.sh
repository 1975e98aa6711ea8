for c in config0 config0 config2 config2; do
  st=2000; [ $c = config2 ] && st=50
  timeout 900 python bench.py --config $c --steps $st --warmup 20 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value']/1e6, 'e2e', d['e2e']['value']/1e6)"
done
