# A-resident vocab argmax GEMM: kernel + parity tests, bench A/B (FNMT_GEMM_AR=0 vs default)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "argmax" > gpurun_out/t_ar_k.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/t_ar_k.log
timeout 900 python -m pytest tests -q -m gpu -x -k "corpus or greedy or smoke or translator" > gpurun_out/t_ar.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_ar.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ar.json 2> gpurun_out/bench_ar.err; echo "bench rc=$?"
FNMT_GEMM_AR=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ar0.json 2> gpurun_out/bench_ar0.err; echo "bench0 rc=$?"
python tools/bsum.py gpurun_out/bench_ar.json gpurun_out/bench_ar0.json
