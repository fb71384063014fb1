# Round-2 evidence pass: traffic/full captures/sanitizers/2-rank dry run
# (gpu_r2_prof.sh) + a serialised launch list of one 3072-row decode batch.
T=${1:-r2e}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/step_launches_$T.csv python tools/perf_step.py 3072 20 1 > gpurun_out/step_$T.log 2>&1
echo "step launches rc=$?"; tail -1 gpurun_out/step_$T.log
python tools/perf_step.py 3072 20 1 >> gpurun_out/step_$T.log 2>&1; tail -1 gpurun_out/step_$T.log
python tools/perf_step.py 3072 20 4 >> gpurun_out/step_$T.log 2>&1; tail -1 gpurun_out/step_$T.log
gzip -f gpurun_out/step_launches_$T.csv
bash tools/gpu_r2_prof.sh $T
