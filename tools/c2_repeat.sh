# config 2: six consecutive bench runs (device and e2e legs)
for i in 1 2 3 4 5 6; do
  timeout 600 python bench.py --config config2 --steps 50 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $i: device %.1f M reads/s (%.2f ms/step), e2e %.1f M' % (d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6))"
done
