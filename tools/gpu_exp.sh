timeout 900 python -m pytest tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py tests/test_gpu_memory.py -q -x -s -m gpu -k "s611 or folded or memory" 2>&1 | grep -E "parity:|passed|failed|assert" | cut -c1-200
python tools/step_live.py 3072 20 | tail -1
FNMT_TOKTAB16=0 python tools/step_live.py 3072 20 | tail -1
bash tools/gpu_ab.sh "FNMT_TOKTAB16=0" "FNMT_TOKTAB16=1" "FNMT_TOKTAB16=0" "FNMT_TOKTAB16=1"
