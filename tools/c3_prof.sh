FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 > gpurun_out/c3_trace.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_inexact_bi -c 2 -o gpurun_out/c3_bi -f python tools/prof_c3.py 200000 1 > gpurun_out/c3_ncu.log 2>&1
ncu -i gpurun_out/c3_bi.ncu-rep --page details --csv > gpurun_out/c3_bi_details.csv 2>&1
