timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in config2 config2 config0 config3; do timeout 1500 python bench.py --config $c --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value']/1e6, 'e2e', d['e2e']['value']/1e6)"; done
