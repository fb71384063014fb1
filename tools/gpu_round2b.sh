mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_corpus_parity.py -q -x -s -m gpu -k "folded or beam" > gpurun_out/t_b.log 2>&1; echo "t rc=$?"
grep -E "parity:|^bf16|^f16|passed|failed" gpurun_out/t_b.log | cut -c1-600
bash tools/gpu_ab.sh "FNMT_DEC_BULK=0" "FNMT_BULK_KB=16" "FNMT_BULK_KB=24" "FNMT_BULK_KB=32" "FNMT_BULK_NT=128 FNMT_BULK_KB=16" "FNMT_BULK_NT=128 FNMT_BULK_KB=24" "FNMT_BULK_NT=128 FNMT_BULK_KB=48" "FNMT_DEC_BULK=0"
