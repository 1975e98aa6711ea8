python -m pytest tests -m gpu -x -q -k "kmer or prefix_table or config4 or scale_golden or config0 or exact" > gpurun_out/t_k.log 2>&1; tail -2 gpurun_out/t_k.log
for k in 12 13 14 15; do echo "=== config4 K=$k"; FMG_LUT_K=$k python tools/prof_exact.py 28 4 2>&1 | grep -E "rep|parity"; done
for k in 13 14; do echo "=== config3 K=$k"; FMG_LUT_K=$k python tools/prof_c3.py 1000000 5 2>&1 | tail -2; done
