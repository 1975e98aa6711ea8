# ncu --set full of the flat z=1 kernels on a config-3-style pass (200k reads = 2.8M seeds, 3.1 Gbp)
mkdir -p gpurun_out
FMG_BIDIR=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_flat_ -c 6 -o gpurun_out/r02_flat -f python tools/prof_c3.py 200000 1 > gpurun_out/flat_ncu.log 2>&1
tail -5 gpurun_out/flat_ncu.log
ls -la gpurun_out/r02_flat.ncu-rep
