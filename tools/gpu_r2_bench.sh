# default bench (kernel profile, parity, cpu baseline) + traffic of the top class
mkdir -p gpurun_out
T=${1:-r2d}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
python - "$T" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
for k in ("value", "e2e", "roofline", "clocks", "gpu_launches"): print(k, json.dumps(d.get(k)))
p = d.get("parity") or {}
print("parity", {k: p.get(k) for k in ("sentences", "identical", "identical_frac", "all_near_ties", "pass")})
print("cpu", json.dumps(d.get("cpu_baseline")))
for k, v in (d.get("kernel_profile") or {}).items(): print(" ", k, v)
PY
export FNMT_LANES=1
timeout 900 ncu --profile-from-start off --cache-control none --clock-control none -k "regex:attn_dec|dec_layer|gemm_tc" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/traffic_$T.csv python tools/profile_traffic.py $T > gpurun_out/traffic_$T.log 2>&1
echo "traffic rc=$?"; tail -1 gpurun_out/traffic_$T.log
python tools/traffic_ratio.py gpurun_out/traffic_$T.csv gpurun_out/prof_log_$T.npz > gpurun_out/traffic_$T.json; cat gpurun_out/traffic_$T.json; gzip -f gpurun_out/traffic_$T.csv
