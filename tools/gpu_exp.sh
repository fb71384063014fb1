timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "attn or attention" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_corpus_parity.py -q -x -m gpu 2>&1 | tail -1
for spc in 0 4; do for L in 12 16 24 32 40; do FNMT_ATTN_SPC=$spc python tools/perf_attn.py $L | sed "s/^/spc=$spc /"; done; done
bash tools/gpu_ab.sh "FNMT_ATTN_SPC=0" "FNMT_ATTN_SPC=4" "FNMT_ATTN_SPC=2" "FNMT_ATTN_SPC=0" "FNMT_ATTN_SPC=4"
