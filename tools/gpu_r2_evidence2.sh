# Round-2 final evidence on the current kernels: bench profile-pass traffic
# (-> profiles/ncu_traffic.json), --set full captures of the top kernels,
# compute-sanitizer memcheck / racecheck, the 2-rank dry run, a launch list.
T=${1:-r2z}
mkdir -p gpurun_out
export FNMT_LANES=1
timeout 900 ncu --profile-from-start off --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/traffic_$T.csv python tools/profile_traffic.py $T > gpurun_out/traffic_$T.log 2>&1
echo "traffic rc=$?"; tail -1 gpurun_out/traffic_$T.log
python tools/traffic_ratio.py gpurun_out/traffic_$T.csv gpurun_out/prof_log_$T.npz > gpurun_out/traffic_$T.json; gzip -f gpurun_out/traffic_$T.csv
for spec in "layer:dec_layer:700:1" "encpipe:attn_enc_pipe:30:1" "norm:add_norm:1000:1" "gemmenc:gemm_tc:0:4" "gemmdec:gemm_tc:1500:4"; do
  IFS=: read name pat skip cnt <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:$pat" \
      --launch-skip $skip --launch-count $cnt -o gpurun_out/full_${T}_$name \
      python tools/profile_traffic.py ${T}_$name > gpurun_out/ncu_full_${T}_$name.log 2>&1
  echo "full $name rc=$?"
done
unset FNMT_LANES
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/step_launches_$T.csv python tools/perf_step.py 3072 20 1 > gpurun_out/step_$T.log 2>&1
echo "launch list rc=$?"; gzip -f gpurun_out/step_launches_$T.csv
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_errors.py tests/test_gpu_parity.py -q -x -m gpu -k "not random" > gpurun_out/memcheck_$T.log 2>&1
echo "memcheck rc=$?"; tail -3 gpurun_out/memcheck_$T.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "attn or decode or norm or embed" > gpurun_out/racecheck_$T.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/racecheck_$T.log
FNMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --profile-sentences 0 > gpurun_out/bench_2rank_$T.json 2> gpurun_out/bench_2rank_$T.err
echo "2rank rc=$?"; head -c 600 gpurun_out/bench_2rank_$T.json
