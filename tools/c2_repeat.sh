# config 2 device leg vs the bench's own clock sampler (nvidia-smi -lms N running during the timed region)
for ms in 100 2000 100 2000 100 2000 100 2000; do
  FMG_BENCH_CLOCK_MS=$ms timeout 600 python bench.py --config config2 --steps 50 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sampler every $ms ms: device %.1f M reads/s (%.2f ms/step), e2e %.1f M, clock samples %d' % (d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['clocks']['samples']))"
done
