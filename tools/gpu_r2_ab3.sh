mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_int8.py tests/test_gpu_beam.py -q -x -m gpu > gpurun_out/t_ab3.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ab3.log
bash tools/gpu_ab.sh "FNMT_BN_WAVE_LONGK=0.15" "FNMT_BN_WAVE_LONGK=0.3" "FNMT_BN_WAVE_LONGK=0.6" "FNMT_BN_WAVE_LONGK=1.0" "FNMT_BN_WAVE_LONGK=0.15" "FNMT_BN_WAVE_LONGK=0.3"
