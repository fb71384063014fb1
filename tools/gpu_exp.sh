timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -3
python tools/perf_gemm.py | tail -5
FNMT_TMA_STORE=0 python tools/perf_gemm.py | tail -5
python tools/perf_gemm.py dec
FNMT_TMA_STORE=0 python tools/perf_gemm.py dec
