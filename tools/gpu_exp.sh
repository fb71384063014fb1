bash tools/gpu_ab.sh "FNMT_GEMM_LN=0" "FNMT_GEMM_LN=1" "FNMT_GEMM_LN=0" "FNMT_GEMM_LN=1"
