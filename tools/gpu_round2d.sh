mkdir -p gpurun_out
python -m pytest tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -s -m gpu -k "greedy or folded or config1" > gpurun_out/t_d.log 2>&1; echo "t rc=$?"
grep -E "parity:|^bf16|^f16|divergences|passed|failed|Error" gpurun_out/t_d.log | cut -c1-400
bash tools/gpu_ab.sh "FNMT_FUSED_SELF=0" "FNMT_FUSED_SELF=1" "FNMT_FUSED_SELF=0" "FNMT_FUSED_SELF=1"
