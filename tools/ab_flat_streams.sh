# flat engine chunk pipeline: streams x queue size (chunk = queue / 48 patterns); config-3-style 14M-seed call
mkdir -p gpurun_out
run() {
  echo "== streams=$1 qcap_log2=$2"
  FMG_FLAT_STREAMS=$1 FMG_FLAT_QCAP_LOG2=$2 FMG_BIDIR=0 FMG_TRACE=1 timeout 900 python tools/prof_c3.py 1000000 4 2>&1 | grep -E "flat z=1|summary|checksum" | tail -2 | cut -c1-260
}
run 3 26
run 4 26
run 3 25
run 4 25
run 4 24
run 2 25
