timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_corpus_parity.py tests/test_gpu_fused_layer.py tests/test_gpu_translator.py tests/test_gpu_kernels.py -q -x -m gpu 2>&1 | tail -1
bash tools/gpu_ab.sh "FNMT_LIVE_ROWS=0" "FNMT_LIVE_ROWS=1" "FNMT_LIVE_ROWS=0" "FNMT_LIVE_ROWS=1"
