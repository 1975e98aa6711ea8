for i in 1 2 3 4; do
  FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline > gpurun_out/c2_var_$i.log 2>&1
  python - $i <<'PY'
import json, sys, re
i = sys.argv[1]
lines = open(f"gpurun_out/c2_var_{i}.log").read().splitlines()
d = json.loads([l for l in lines if l.startswith("{")][-1])
print(i, "ms/step", round(d["ms_per_step"], 2), "clocks", d["clocks"])
tr = [l for l in lines if "split" in l]
for l in tr[3:9]: print("   ", l[:170])
PY
done
