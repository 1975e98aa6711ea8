# Full GPU evidence pass: tests, every config through bench.py (+ reference arm), ncu captures.
set -x
(time timeout 2400 python -m pytest tests -m gpu -q) > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/bench_all.sh > gpurun_out/bench_all_summary.txt 2>&1; cat gpurun_out/bench_all_summary.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_occ_pair -s 3 -c 1 -o gpurun_out/r02_occ_config1 -f python tools/prof_occ.py config1 > gpurun_out/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact -s 1 -c 1 -o gpurun_out/r02_c4_exact -f python tools/prof_exact.py 24 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep
bash tools/flat_check.sh > gpurun_out/flat_check.log 2>&1; tail -4 gpurun_out/flat_check.log | cut -c1-200
bash tools/flat_prof.sh
