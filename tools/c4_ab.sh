timeout 900 python -m pytest tests -m gpu -x -q -k "kmer or exact or config4" 2>&1 | tail -2
for v in "FMG_X=0" "FMG_EXACT_LUT_EXT=0"; do
  env $v timeout 900 python bench.py --config config4 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value']/1e9, 'G seeds/s', d['ms_per_step'], d.get('kmer_table'), d.get('roofline',{}).get('frac'), d['e2e']['value']/1e9)"
done
timeout 900 python bench.py --config config0 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-250
