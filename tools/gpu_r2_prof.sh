# Round-2 evidence: per-launch DRAM traffic of the bench's profile pass matched
# against the engine's algorithmic counts, --set full captures of the top
# kernels, compute-sanitizer memcheck / racecheck, a 2-rank dry run of bench.
T=${1:-r2a}
mkdir -p gpurun_out
export FNMT_LANES=1
timeout 900 ncu --profile-from-start off --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/traffic_$T.csv python tools/profile_traffic.py $T > gpurun_out/traffic_$T.log 2>&1
echo "traffic rc=$?"; tail -2 gpurun_out/traffic_$T.log
python tools/traffic_ratio.py gpurun_out/traffic_$T.csv gpurun_out/prof_log_$T.npz > gpurun_out/traffic_$T.json; cat gpurun_out/traffic_$T.json
gzip -f gpurun_out/traffic_$T.csv
for spec in "attn_dec:regex:dec_layer:700:2" "attn_enc:regex:attn_enc_pipe:60:2" "norm:regex:add_norm:1000:2" \
            "gemm:regex:gemm_tc:1500:8"; do
  IFS=: read name kind pat skip cnt <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "$kind:$pat" \
      --launch-skip $skip --launch-count $cnt -o gpurun_out/full_${T}_$name \
      python tools/profile_traffic.py ${T}_$name > gpurun_out/ncu_full_${T}_$name.log 2>&1
  echo "full $name rc=$?"
  ncu -i gpurun_out/full_${T}_$name.ncu-rep --page raw --csv > gpurun_out/full_${T}_$name.csv 2>/dev/null
  gzip -f gpurun_out/full_${T}_$name.csv
done
unset FNMT_LANES
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_errors.py -q -x -m gpu > gpurun_out/memcheck_$T.log 2>&1
echo "memcheck rc=$?"; tail -4 gpurun_out/memcheck_$T.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "attn or decode or norm or embed" > gpurun_out/racecheck_$T.log 2>&1
echo "racecheck rc=$?"; tail -4 gpurun_out/racecheck_$T.log
FNMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --profile-sentences 0 > gpurun_out/bench_2rank_$T.json 2> gpurun_out/bench_2rank_$T.err
echo "2rank rc=$?"; head -c 3000 gpurun_out/bench_2rank_$T.json; tail -3 gpurun_out/bench_2rank_$T.err
