mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_layer.py tests/test_gpu_corpus_parity.py -q -x -s -m gpu -k "not greedy_update" > gpurun_out/t_l2.log 2>&1; echo "tests rc=$?"
grep -E "parity:|identical|passed|failed|Error|assert" gpurun_out/t_l2.log | cut -c1-300 | tail -10
python tools/step_live.py 3072 20
python tools/step_live.py 1536 40 | head -2
bash tools/gpu_ab.sh "FNMT_LANES=4" "FNMT_LANES=4"
