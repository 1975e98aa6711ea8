# config 1 Occ kernel: neighbouring lanes fetching each other's lines (one request per step's two lines when they share a 128-byte block)
FMG_OCC_EXCH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config1 or occ" 2>&1 | tail -2
for v in 0 1 0 1; do FMG_OCC_EXCH=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-hbm-extra 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exch=$v device %.4g steps/s (%.4f ms) frac %s' % (d['value'], d['ms_per_step'], d['roofline']['frac']))"; done
