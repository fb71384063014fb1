mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused_layer.py -q -x -m gpu > gpurun_out/t_ab1.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ab1.log
bash tools/gpu_ab.sh "FNMT_LANES=4" "FNMT_LAYER_NT=256" "FNMT_LAYER_KB=12" "FNMT_LAYER_KB=24" "FNMT_GEMM_DUAL=0" "FNMT_BN_WAVE=0.3" "FNMT_LANES=6" "FNMT_LANES=4"
