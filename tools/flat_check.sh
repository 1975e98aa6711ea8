# flat z=1 engine: parity tests, then the config-3-style pass (14M seeds, 3.1 Gbp) with the trace,
# presence filter off and on (same checksum expected)
mkdir -p gpurun_out
(timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "flat or config3_small" 2>&1 | tail -15) > gpurun_out/flat_tests.log 2>&1
cat gpurun_out/flat_tests.log
FMG_FLAT_FILTER=0 FMG_BIDIR=0 FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | tail -12 | tee gpurun_out/flat_filter_off.log
FMG_BIDIR=0 FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 4 2>&1 | tail -20 | tee gpurun_out/flat_filter_on.log
