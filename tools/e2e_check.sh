for i in 1 2; do
FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c2_tr.log 2>&1
grep "^{" gpurun_out/c2_tr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config2', d['value']/1e6, 'e2e', d['e2e']['value']/1e6)"
grep "z1 bidir" gpurun_out/c2_tr.log | sed 's/.*spines+chains \([0-9.]*\) ms.*dedup\/sort \([0-9.]*\) ms.*/\1+\2/' | tr '\n' ' '; echo
done
