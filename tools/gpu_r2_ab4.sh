mkdir -p gpurun_out
for env in "FNMT_GEMM_SMALLM=1" "FNMT_GEMM_SMALLM=2" "FNMT_SPLITK=4"; do
  env $env timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_corpus_parity.py -q -x -m gpu -k "not beam" > gpurun_out/t_ab4.log 2>&1; echo "tests [$env] rc=$?"; tail -1 gpurun_out/t_ab4.log
done
bash tools/gpu_ab.sh "FNMT_GEMM_SMALLM=0" "FNMT_GEMM_SMALLM=1" "FNMT_GEMM_SMALLM=2" "FNMT_SPLITK=2" "FNMT_SPLITK=4" "FNMT_GEMM_SMALLM=1 FNMT_SPLITK=4" "FNMT_GEMM_SMALLM=0" "FNMT_GEMM_SMALLM=1"
