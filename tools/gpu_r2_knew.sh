mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/t_knew.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_knew.log
python tools/step_live.py 3072 20
FNMT_KNEW_STAGE=0 python tools/step_live.py 3072 20
bash tools/gpu_ab.sh "FNMT_KNEW_STAGE=0" "FNMT_KNEW_STAGE=1" "FNMT_KNEW_STAGE=0" "FNMT_KNEW_STAGE=1"
