mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -q -x) > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in config2 config3; do
  steps=50; [ $c = config3 ] && steps=2
  (time timeout 1500 python bench.py --config $c --steps $steps --warmup 3 --no-hbm-extra) 2>gpurun_out/bench_$c.err | tail -1 > gpurun_out/bench_$c.json
  tail -4 gpurun_out/bench_$c.err; cut -c1-400 gpurun_out/bench_$c.json
done
