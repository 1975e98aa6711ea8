#!/bin/bash
# A/B of library builds in tools/ab/*.so on one workload script.
# usage: bash tools/ab_run.sh "<python script + args>" lib1 lib2 ...   (FMG_TRACE=1 per-kernel timings)
cmd=$1; shift
for lib in "$@"; do
  echo "=== $lib"
  FMG_TRACE=1 FMG_LIB_PATH=tools/ab/$lib.so timeout 600 python $cmd 2>&1 | tail -8
done
