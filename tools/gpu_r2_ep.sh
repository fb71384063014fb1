# argmax epilogue: two TMEM loads per wait — kernel + parity tests, bench A/B on one box
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "argmax or linear" > gpurun_out/t_ep_k.log 2>&1; echo "kernel tests rc=$?"; tail -1 gpurun_out/t_ep_k.log
timeout 900 python -m pytest tests -q -m gpu -x -k "corpus or greedy" > gpurun_out/t_ep.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_ep.log
for cfg in "ep1:" "ep0:FNMT_ARGMAX_PAIRS=0" "ep1b:" "ep0b:FNMT_ARGMAX_PAIRS=0"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ep_$tag.json 2> gpurun_out/ep_$tag.err; echo "$tag rc=$?"
done
python tools/bsum.py gpurun_out/ep_*.json 2>&1 | grep -v "^   [a-uw-z]"
