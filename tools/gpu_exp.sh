timeout 900 python -m pytest tests/test_gpu_beam.py tests/test_gpu_corpus_parity.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -2
timeout 1200 python bench.py --model 6-6-8 --beam 4 --profile-sentences 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4c.json 2>/dev/null
timeout 1200 python bench.py --model deep-12-768 --dtype bf16 --beam 4 --profile-sentences 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5c.json 2>/dev/null
for f in cfg4c cfg5c; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['kernel_profile']['vocab_argmax'])"; done
export FNMT_LANES=1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:gemm_tc_kernel<\(int\)256, \(int\)4, \(int\)4" --launch-skip 10 --launch-count 1 \
  -o gpurun_out/full_r2j_topk python tools/profile_traffic.py r2j_topk 1024 6-6-8 4 f16 > gpurun_out/ncu_r2j_topk.log 2>&1; echo "topk rc=$?"
