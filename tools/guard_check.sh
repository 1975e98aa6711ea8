#!/bin/bash
# The GPU test suite under guard mode (FMG_GUARD=1: every library allocation ends at an unmapped
# guard page, so any out-of-bounds read or write of index lines, chunks, tables, scratch or
# results faults).  compute-sanitizer is not available on this GPU pool.
out=gpurun_out
FMG_GUARD=1 timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider \
  --deselect tests/test_gpu_scale.py --deselect tests/test_gpu_multirank.py::test_bench_self_launches_two_ranks \
  > $out/guard_check.log 2>&1
echo "guard_check rc=$?" >> $out/guard_check.log
tail -3 $out/guard_check.log
