mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py tests/test_gpu_translator.py -q -x -s -m gpu > gpurun_out/t_tab.log 2>&1; echo "tests rc=$?"
grep -E "parity:|identical|passed|failed|Error|assert" gpurun_out/t_tab.log | cut -c1-300 | tail -14
python tools/step_live.py 3072 20
python tools/step_live.py 1536 40 | head -2
bash tools/gpu_ab.sh "FNMT_STEP_TABLES=0" "FNMT_STEP_TABLES=1" "FNMT_STEP_TABLES=0" "FNMT_STEP_TABLES=1"
