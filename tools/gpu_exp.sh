timeout 900 python -m pytest tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -s -m gpu -k "s611 or folded" 2>&1 | grep -E "parity:|passed|failed|assert|Error" | cut -c1-250
for u in 2 3 4; do FNMT_LAYER_U=$u python tools/step_live.py 3072 20 | sed -n 2p | sed "s/^/U=$u 3072 /"; FNMT_LAYER_U=$u python tools/step_live.py 1536 40 | sed -n 2p | sed "s/^/U=$u 1536 /"; done
FNMT_LAYER_REG=0 python tools/step_live.py 3072 20 | sed -n 2p | sed "s/^/ring 3072 /"
bash tools/gpu_ab.sh "FNMT_LAYER_REG=0" "FNMT_LAYER_REG=1" "FNMT_LAYER_REG=1 FNMT_LAYER_U=2" "FNMT_LAYER_REG=0" "FNMT_LAYER_REG=1"
