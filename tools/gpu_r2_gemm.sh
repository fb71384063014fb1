# decoder GEMM shapes under the small-M variants
mkdir -p gpurun_out
for v in 0 1 2; do echo "FNMT_GEMM_SMALLM=$v"; FNMT_GEMM_SMALLM=$v python tools/perf_gemm.py dec; done
for w in 0.15 0.6 2; do echo "FNMT_BN_WAVE=$w"; FNMT_BN_WAVE=$w python tools/perf_gemm.py dec; done
