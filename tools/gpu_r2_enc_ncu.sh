mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/t_k.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_k.log
export FNMT_LANES=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 0 --launch-count 5 \
  -o gpurun_out/full_r2g_enc python tools/profile_traffic.py r2g_enc 8192 > gpurun_out/ncu_r2g_enc.log 2>&1; echo "enc rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel.*256,.4,.4 --launch-skip 30 --launch-count 2 \
  -o gpurun_out/full_r2g_topk python tools/profile_traffic.py r2g_topk 1024 6-6-8 4 f16 > gpurun_out/ncu_r2g_topk.log 2>&1; echo "topk rc=$?"
tail -3 gpurun_out/ncu_r2g_topk.log
