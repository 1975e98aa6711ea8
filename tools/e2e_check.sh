FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c2_tr.log 2>&1
grep "^{" gpurun_out/c2_tr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config2', d['value']/1e6, 'e2e', d['e2e']['value']/1e6)"
grep "\[fmg\]" gpurun_out/c2_tr.log | sed -n 20,40p | cut -c1-150
