for i in 1 2 3; do
FMG_TRACE=1 timeout 600 python bench.py --config config2 --steps 50 --warmup 10 --no-hbm-extra --no-cpu-baseline > gpurun_out/c2d.log 2>&1
grep "^{" gpurun_out/c2d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config2', d['value']/1e6, d['ms_per_step'])"
grep "z1 bidir" gpurun_out/c2d.log | sed -n 11,60p | sed 's/.*spines+chains \([0-9.]*\) ms.*dedup\/sort \([0-9.]*\) ms.*/\1 \2/' | awk '{a+=$1; b+=$2; if ($1>m) m=$1} END {print "mean spines+chains", a/NR, "max", m, "mean dedup", b/NR}'
grep "fmg_inexact host time" gpurun_out/c2d.log | sed -n 11,60p | sed 's/.*validate \([0-9.]*\) ms, search \([0-9.]*\) ms/\1 \2/' | awk '{a+=$1; b+=$2; if ($2>m) m=$2} END {print "mean validate", a/NR, "mean search", b/NR, "max search", m}'
grep "pre-engine" gpurun_out/c2d.log | sed -n 11,60p | sed 's/.*time \([0-9.]*\) ms/\1/' | awk '{a+=$1; if ($1>m) m=$1} END {print "mean pre-engine", a/NR, "max", m}'
done
