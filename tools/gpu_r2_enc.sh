# pipelined encoder attention: tests, A/B, ncu capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_corpus_parity.py -q -x -s -m gpu > gpurun_out/t_enc.log 2>&1; echo "tests rc=$?"
grep -E "parity:|passed|failed|Error" gpurun_out/t_enc.log | cut -c1-200 | tail -8
bash tools/gpu_ab.sh "FNMT_ATTN_PIPE=0" "FNMT_ATTN_PIPE=1" "FNMT_ATTN_PIPE=0" "FNMT_ATTN_PIPE=1"
export FNMT_LANES=1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:attn_enc_pipe" \
      --launch-skip 60 --launch-count 2 -o gpurun_out/full_r2c_enc python tools/profile_traffic.py r2c_enc > gpurun_out/ncu_full_r2c_enc.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/full_r2c_enc.ncu-rep --page raw --csv > gpurun_out/full_r2c_enc.csv 2>/dev/null; gzip -f gpurun_out/full_r2c_enc.csv
python tools/ncu_metrics.py gpurun_out/full_r2c_enc.csv.gz | cut -c1-200
