#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root):
#   1. launch list with per-launch duration and DRAM bytes of a fixed
#      workload (profile_step: 2048 newstest-shaped sentences, 6-1-1 fp16,
#      one decode lane so the launch order is phase-ordered);
#   2. --set full captures of the decode GEMM, vocab GEMM, decode attention,
#      encoder attention and add+LayerNorm kernels, exported as raw CSV.
# Output under gpurun_out/ (raw-page CSVs gzipped; the .ncu-rep files are dropped).
set -u
R=${1:-r1}
mkdir -p gpurun_out
export FNMT_LANES=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python tools/profile_step.py 2048 > gpurun_out/ncu_launches_$R.log 2>&1
gzip -f gpurun_out/launches_$R.csv
# ncu -k matches the base kernel name (no template arguments): 7 consecutive
# GEMMs from launch 100 on are one full decode step (6 decoder GEMMs + vocab).
for spec in "gemm_step:regex:gemm_tc:100:7" "attn_dec:regex:attn_decode:200:2" \
            "attn_enc:regex:attn_varlen:4:1" "norm:regex:add_norm:300:2"; do
  IFS=: read name kind pat skip cnt <<< "$spec"
  ncu --set full --clock-control none --import-source on -k "$kind:$pat" --launch-skip $skip \
      --launch-count $cnt -o gpurun_out/full_${R}_$name \
      python tools/profile_step.py 2048 > gpurun_out/ncu_full_${R}_$name.log 2>&1
  ncu -i gpurun_out/full_${R}_$name.ncu-rep --page raw --csv > gpurun_out/full_${R}_$name.csv 2>/dev/null
  gzip -f gpurun_out/full_${R}_$name.csv
  sz=$(stat -c %s gpurun_out/full_${R}_$name.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 0 ]; then rm -f gpurun_out/full_${R}_$name.ncu-rep; fi
done
ls -la gpurun_out
