mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -s -m gpu > gpurun_out/t_mma.log 2>&1; echo "tests rc=$?"
grep -E "parity:|identical|passed|failed|Error|assert" gpurun_out/t_mma.log | cut -c1-400 | tail -14
python tools/step_live.py 3072 20
python tools/step_live.py 1536 40
FNMT_LAYER_STAGES=6 python tools/step_live.py 1536 40
FNMT_LAYER_MMA=0 python tools/step_live.py 1536 40
bash tools/gpu_ab.sh "FNMT_LAYER_MMA=0" "FNMT_LAYER_MMA=1" "FNMT_LAYER_MMA=0" "FNMT_LAYER_MMA=1"
