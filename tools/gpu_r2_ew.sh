# vocab argmax GEMM with 16 epilogue warps: argmax tests, corpus parity, bench A/B (FNMT_ARGMAX_EW16=0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "argmax" > gpurun_out/t_ew_k.log 2>&1; echo "kernel tests rc=$?"; tail -1 gpurun_out/t_ew_k.log
timeout 900 python -m pytest tests -q -m gpu -x -k "corpus or greedy" > gpurun_out/t_ew.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_ew.log
for cfg in "e16:" "e8:FNMT_ARGMAX_EW16=0" "e16b:" "e8b:FNMT_ARGMAX_EW16=0"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ew_$tag.json 2> gpurun_out/ew_$tag.err; echo "$tag rc=$?"
done
python tools/bsum.py gpurun_out/ew_*.json 2>&1 | grep -v "^   [a-uw-z]"
