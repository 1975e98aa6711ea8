#!/bin/bash
# Every BASELINE config through bench.py (our arm + the reference arm); JSON lines into gpurun_out/bench_all.jsonl
mkdir -p gpurun_out
out=gpurun_out/bench_all.jsonl
: > $out
for c in config1 config0 config2 config1h config4 config3; do
  sleep 10  # the previous process has released its device memory before this one sizes its scratch
  # enough steps for a timed region of tens of ms (config 0 steps are ~12 us each)
  steps=10; [ $c = config3 ] && steps=2; [ $c = config0 ] && steps=2000; [ $c = config2 ] && steps=50
  timeout 1500 python bench.py --config $c --steps $steps --warmup 3 --no-hbm-extra 2>gpurun_out/bench_$c.err | tail -1 >> $out
  timeout 2400 python bench.py --impl reference --config $c --steps 3 --warmup 3 2>gpurun_out/ref_$c.err | tail -1 >> $out
done
python - <<'PY'
import json
for line in open("gpurun_out/bench_all.jsonl"):
    try:
        d = json.loads(line)
    except Exception:
        continue
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    c = d.get("cpu_baseline") or {}
    print(f"{d.get('impl','ours'):9s} {d['config']['workload'][:40]:40s} value={d['value']:.4g} {d['unit']} "
          f"e2e={e.get('value', 0):.4g} frac={r.get('frac')} cpu={c.get('value', 0):.4g}")
PY
