# config 2 device-path stability: the exact bench_all prefix (config 1 and 0, both arms), then config 2 with the trace
for c in config1 config0; do
  sleep 10
  steps=10; [ $c = config0 ] && steps=2000
  timeout 1500 python bench.py --config $c --steps $steps --warmup 3 --no-hbm-extra 2>/dev/null | tail -1 | cut -c1-120
  timeout 2400 python bench.py --impl reference --config $c --steps 3 --warmup 3 2>/dev/null | tail -1 | cut -c1-120
done
sleep 10
for i in 1 2; do
  FMG_TRACE=$((i-1)) ; [ $i = 1 ] && unset FMG_TRACE || export FMG_TRACE=1
  timeout 600 python bench.py --config config2 --steps 50 --warmup 3 --no-hbm-extra 2>gpurun_out/c2_trace_$i.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $i: device %.1f M reads/s (%.2f ms/step), e2e %.1f M, clock samples %d' % (d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['clocks']['samples']))"
  grep "z1 bidirectional" gpurun_out/c2_trace_$i.err | sed -E 's/.*spines\+chains ([0-9.]+) ms, group\/sort\/dedup ([0-9.]+) ms.*/\1 \2/' | awk '{a[NR]=$1; b[NR]=$2; s+=$1; t+=$2} END {if (NR) print "   calls", NR, "mean spines+chains", s/NR, "mean group/sort/dedup", t/NR}'
done
