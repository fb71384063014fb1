# vocab argmax GEMM: L2 prefetch of the next W tile — argmax tests, corpus parity, bench A/B (FNMT_W_PREFETCH=0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "argmax" > gpurun_out/t_pf_k.log 2>&1; echo "kernel tests rc=$?"; tail -1 gpurun_out/t_pf_k.log
timeout 900 python -m pytest tests -q -m gpu -x -k "corpus or greedy" > gpurun_out/t_pf.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_pf.log
for cfg in "p1:" "p0:FNMT_W_PREFETCH=0" "p1b:" "p0b:FNMT_W_PREFETCH=0"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pf_$tag.json 2> gpurun_out/pf_$tag.err; echo "$tag rc=$?"
done
python tools/bsum.py gpurun_out/pf_*.json 2>&1 | grep -v "^   [a-uw-z]"
