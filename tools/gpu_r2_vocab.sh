# --set full capture of the vocab argmax GEMM over the bench profile pass
mkdir -p gpurun_out
FNMT_LANES=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:gemm_tc_kernel<\(int\)256, \(int\)4, \(int\)0, \(bool\)0, \(int\)1, \(int\)2, \(bool\)0>" --launch-skip 300 --launch-count 2 \
  -o gpurun_out/full_r2v_vocab python tools/profile_traffic.py r2v_vocab > gpurun_out/ncu_full_r2v_vocab.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full_r2v_vocab.log
