timeout 900 python -m pytest tests -m gpu -x -q -k "bidirectional or z1 or repeated or inexact or config3" 2>&1 | tail -2
for v in "FMG_X=0" "FMG_BI_JUMPX=0"; do
  echo "=== $v"
  env $v FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 3 2>&1 | grep "split\|summary" | tail -2 | cut -c1-150
done
