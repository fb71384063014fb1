# decoder residual + norm fused into the o-proj / FFN2 GEMM: tests, bench A/B (FNMT_NORM_FUSE=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "norm or corpus or greedy or beam or memory or linear or s618" > gpurun_out/t_nf.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_nf.log
for cfg in "nf1:" "nf0:FNMT_NORM_FUSE=0" "nf1b:" "nf0b:FNMT_NORM_FUSE=0"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 600 python bench.py --no-cpu-baseline > gpurun_out/nf_$tag.json 2> gpurun_out/nf_$tag.err; echo "$tag rc=$?"
done
for cfg in "m1:" "m0:FNMT_NORM_FUSE=0"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 900 python bench.py --model 6-1-8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nf_$tag.json 2> gpurun_out/nf_$tag.err; echo "$tag rc=$?"
done
python tools/bsum.py gpurun_out/nf_*.json 2>&1 | grep -v "^   [a-fh-mo-uw-z]"
