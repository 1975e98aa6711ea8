# config 1-H (1 Gbp, HBM-resident Occ steps): 128-byte chunks vs 64-byte chunks (adaptive-width loads, and
# every load hinted 64 B: tools/ab/nowide.so built with -DFMG_CHUNK2_WIDE=0)
mkdir -p gpurun_out
run() {  # label, sectors, lib
  FMG_CHUNK_SECTORS=$2 FMG_LIB_PATH=$3 timeout 900 python bench.py --config config1h --steps 20 --warmup 5 --no-cpu-baseline 2>gpurun_out/ab_1h_$1.err | tail -1 > gpurun_out/ab_1h_$1.jsonl
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_1h_$1.jsonl").read())
r = d["roofline"]
print("$1 value=%.4g e2e=%.4g frac=%s kernel=%s req=%s" % (d["value"], d["e2e"]["value"], r.get("frac"), r.get("kernel"), (r.get("request_roofline") or {}).get("frac")))
PY
}
run chunk4 4 paper_1811_06127_b200/libfmgpu.so
run chunk2_wide 2 paper_1811_06127_b200/libfmgpu.so
[ -f tools/ab/nowide.so ] && run chunk2_hint64 2 tools/ab/nowide.so
