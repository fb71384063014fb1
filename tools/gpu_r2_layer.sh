# fused decoder layer kernel: tests, parity, A/B, traffic of the attention class
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -s -m gpu > gpurun_out/t_layer.log 2>&1; echo "tests rc=$?"
grep -E "parity:|identical|passed|failed|Error" gpurun_out/t_layer.log | cut -c1-300 | tail -20
bash tools/gpu_ab.sh "FNMT_FUSED_LAYER=0" "FNMT_FUSED_LAYER=1" "FNMT_FUSED_LAYER=0" "FNMT_FUSED_LAYER=1"
export FNMT_LANES=1
timeout 900 ncu --profile-from-start off --cache-control none --clock-control none -k "regex:attn_dec|dec_layer" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/traffic_r2b.csv python tools/profile_traffic.py r2b > gpurun_out/traffic_r2b.log 2>&1
echo "traffic rc=$?"; tail -2 gpurun_out/traffic_r2b.log
python tools/traffic_ratio.py gpurun_out/traffic_r2b.csv gpurun_out/prof_log_r2b.npz; gzip -f gpurun_out/traffic_r2b.csv
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:dec_layer" \
      --launch-skip 700 --launch-count 2 -o gpurun_out/full_r2b_layer python tools/profile_traffic.py r2b_layer > gpurun_out/ncu_full_r2b_layer.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/full_r2b_layer.ncu-rep --page raw --csv > gpurun_out/full_r2b_layer.csv 2>/dev/null; gzip -f gpurun_out/full_r2b_layer.csv
