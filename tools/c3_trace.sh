for v in "FMG_X=0" "FMG_POOL_RESERVE_GB=0"; do
env $v FMG_TRACE=1 timeout 1500 python bench.py --config config3 --steps 4 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c3_trace3.log 2>&1
grep "^{" gpurun_out/c3_trace3.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c3', d['value']/1e6, 'e2e', d['e2e']['value']/1e6, d['ms_per_step'])"
grep "split" gpurun_out/c3_trace3.log | sed 's/.*B sort + merge \([0-9.]*\) ms.*/\1/' | tr '\n' ' '; echo
done
