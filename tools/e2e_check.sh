timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in config0 config0 config4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value']/1e6, 'e2e', d['e2e']['value']/1e6, d.get('kmer_table'))"; done
