timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
python tools/perf_gemm.py > /tmp/a.txt; tail -4 /tmp/a.txt
FNMT_TMA_STORE_SINGLE=0 python tools/perf_gemm.py > /tmp/b.txt; tail -4 /tmp/b.txt
