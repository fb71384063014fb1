mkdir -p gpurun_out
T=${1:-r2f}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dec_layer --launch-skip 20 --launch-count 1 \
  -o gpurun_out/full_${T}_layer python tools/step_live.py 3072 20 > gpurun_out/ncu_${T}_layer.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_${T}_layer.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 40 --launch-count 6 \
  -o gpurun_out/full_${T}_gemm python tools/step_live.py 3072 20 > gpurun_out/ncu_${T}_gemm.log 2>&1
echo "rc=$?"
