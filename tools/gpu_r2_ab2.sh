mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_parity.py tests/test_gpu_beam.py -q -x -s -m gpu > gpurun_out/t_ab2.log 2>&1; echo "tests rc=$?"; grep -E "identical|passed|failed" gpurun_out/t_ab2.log | tail -6
bash tools/gpu_ab.sh "FNMT_GREEDY_EMBED=0" "FNMT_GREEDY_EMBED=1" "FNMT_BN_WAVE=0.3" "FNMT_BN_WAVE=0.15" "FNMT_BN_WAVE=0.3 FNMT_LANES=6" "FNMT_BN_WAVE=0.3 FNMT_LANES=5" "FNMT_BN_WAVE=0.3 FNMT_LANES=8" "FNMT_GREEDY_EMBED=0" "FNMT_GREEDY_EMBED=1"
