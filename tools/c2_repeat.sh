# config 2 device-path stability: the bench three times in a row after a large-memory process, trace on the last
timeout 600 python bench.py --config config1h --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for i in 1 2 3; do
  timeout 600 python bench.py --config config2 --steps 50 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $i: device %.1f M reads/s (%.2f ms/step), e2e %.1f M' % (d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6))"
done
FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 20 --warmup 3 2>&1 | grep -E "z1 bidirectional|pre-engine" | awk '{print}' | tail -46 | cut -c1-200 > gpurun_out/c2_trace.log
grep -c "z1 bidirectional" gpurun_out/c2_trace.log; grep "z1 bidirectional" gpurun_out/c2_trace.log | sed -E 's/.*spines\+chains ([0-9.]+) ms, group\/sort\/dedup ([0-9.]+) ms.*/\1 \2/' | sort -n | awk '{a[NR]=$1; b[NR]=$2} END {print "spines+chains min/median/max:", a[1], a[int((NR+1)/2)], a[NR]}'
