timeout 900 python -m pytest tests -m gpu -x -q -k "exact or kmer or config0 or golden" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config config0 --steps 50 --warmup 5 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-150; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c0.csv python bench.py --config config0 --steps 5 --warmup 3 --no-hbm-extra --no-cpu-baseline > /dev/null 2>&1
grep k_exact gpurun_out/launches_c0.csv | tail -3 | cut -c1-300
timeout 600 python bench.py --config config4 --steps 10 --warmup 3 --no-hbm-extra --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-150
