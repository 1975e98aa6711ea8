# config 2 device-path stability: after the GPU test suite (as in tools/round_check.sh), then the bench_all prefix
(timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_scale.py 2>&1 | tail -1)
nvidia-smi --query-compute-apps=pid,used_memory --format=csv,noheader | head -5
for c in config1 config0; do
  sleep 10
  steps=10; [ $c = config0 ] && steps=2000
  timeout 1500 python bench.py --config $c --steps $steps --warmup 3 --no-hbm-extra 2>/dev/null | tail -1 | cut -c1-100
  timeout 2400 python bench.py --impl reference --config $c --steps 3 --warmup 3 2>/dev/null | tail -1 | cut -c1-100
done
sleep 10
nvidia-smi --query-compute-apps=pid,used_memory --format=csv,noheader | head -5
for i in 1 2; do
  timeout 600 python bench.py --config config2 --steps 50 --warmup 3 --no-hbm-extra 2>gpurun_out/c2_trace_$i.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $i: device %.1f M reads/s (%.2f ms/step), e2e %.1f M, clock samples %d, free %.1f GB' % (d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['clocks']['samples'], d['gpu_mem_free_after_index']/1e9))"
done
