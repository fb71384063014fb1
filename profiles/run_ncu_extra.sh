#!/bin/bash
# --set full captures of the kernels profiles/run_ncu.sh does not cover:
# embedding, greedy update, the int8 path (min/max, quantize, kind::i8 GEMM)
# and the beam kernels.  Raw-page CSVs (gzipped) under gpurun_out/.
set -u
R=${1:-r1e}
mkdir -p gpurun_out
export FNMT_LANES=1
run() {  # name kernel-regex skip count profile_step-args...
  local name=$1 pat=$2 skip=$3 cnt=$4; shift 4
  ncu --set full --clock-control none -k "regex:$pat" --launch-skip $skip --launch-count $cnt \
      -o gpurun_out/full_${R}_$name python tools/profile_step.py "$@" \
      > gpurun_out/ncu_full_${R}_$name.log 2>&1
  ncu -i gpurun_out/full_${R}_$name.ncu-rep --page raw --csv > gpurun_out/full_${R}_$name.csv 2>/dev/null
  gzip -f gpurun_out/full_${R}_$name.csv
  rm -f gpurun_out/full_${R}_$name.ncu-rep
}
run embed embed_kernel 40 2 2048 f16
run greedy greedy_update 40 2 2048 f16
run int8 "q_minmax|q_quant|gemm_tc" 200 6 1024 int8
run beam "beam_|gemm_tc_kernel" 100 6 1024 f16 4
ls -la gpurun_out | grep $R
