# config 1 e2e (fmg_occ_pair_host pipeline): chunk size of the H2D / kernel / D2H pipeline
for c in 21 20 19 18 22; do
  FMG_OCC_HOST_CHUNK_LOG2=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-hbm-extra 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk 2^$c: e2e %.4g steps/s, device %.4g' % (d['e2e']['value'], d['value']))"
done
