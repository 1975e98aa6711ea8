#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the GPU tests of every
# kernel family (small inputs).  Logs in gpurun_out/sanitize_*.log; summary lines at the end.
set -u
out=gpurun_out
SEL_MEM="tests/test_gpu_parity.py::test_small_cases_all_paths tests/test_gpu_parity.py::test_acag_occ_api tests/test_gpu_parity.py::test_acag_search_api tests/test_gpu_parity.py::test_exact_edge_cases tests/test_gpu_parity.py::test_inexact_random_vs_oracle tests/test_gpu_parity.py::test_records_and_hits tests/test_gpu_parity.py::test_reconstruct_round_trip tests/test_gpu_parity.py::test_device_pattern_validation_errors tests/test_gpu_buckets.py tests/test_gpu_chunks.py::test_chunk_layout_device_status"
SEL_BI="tests/test_gpu_parity.py::test_inexact_bidirectional_engine tests/test_gpu_parity.py::test_inexact_prefix_table_paths tests/test_gpu_parity.py::test_inexact_repeated_calls_reuse_dedup_table"
run() {  # tool, name, selection
  timeout 3000 compute-sanitizer --tool "$1" --error-exitcode 99 --print-limit 50 --target-processes all \
    python -m pytest -x -q -p no:cacheprovider $3 > "$out/sanitize_$2.log" 2>&1
  echo "$2 rc=$?" >> "$out/sanitize_summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" "$out/sanitize_$2.log" | tail -3 >> "$out/sanitize_summary.txt"
}
: > "$out/sanitize_summary.txt"
run memcheck memcheck "$SEL_MEM"
run memcheck memcheck_bidir "$SEL_BI"
run racecheck racecheck_bidir "$SEL_BI"
run racecheck racecheck_small "tests/test_gpu_parity.py::test_small_cases_all_paths tests/test_gpu_parity.py::test_inexact_random_vs_oracle"
run synccheck synccheck "tests/test_gpu_parity.py::test_small_cases_all_paths tests/test_gpu_parity.py::test_inexact_random_vs_oracle"
run initcheck initcheck "tests/test_gpu_parity.py::test_small_cases_all_paths tests/test_gpu_buckets.py::test_figure2_counts"
cat "$out/sanitize_summary.txt"
