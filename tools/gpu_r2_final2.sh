# Round-2 final record on the final kernels (re-entry session): every GPU test,
# smoke, the default bench (CPU reference arm, parity leg), the reference arm,
# BASELINE configs 3-5, the ncu launch list of the bench command.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1800 python -m pytest tests -q -m gpu -rs -s > gpurun_out/t_final2.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/t_final2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final2.log
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final2.json 2> gpurun_out/bench_ref_final2.err; echo "ref rc=$?"
timeout 900 python bench.py --model 6-1-8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3g.json 2>/dev/null; echo "cfg3 rc=$?"
timeout 1500 python bench.py --model 6-6-8 --beam 4 --profile-sentences 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4g.json 2>/dev/null; echo "cfg4 rc=$?"
timeout 1500 python bench.py --model deep-12-768 --dtype bf16 --beam 4 --profile-sentences 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5g.json 2>/dev/null; echo "cfg5 rc=$?"
cat gpurun_out/cfg3g.json gpurun_out/cfg4g.json gpurun_out/cfg5g.json > gpurun_out/configs_final2.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_final2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_final2.log 2>&1
echo "launch list rc=$?"
python tools/bsum.py gpurun_out/bench_final2.json
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final2.json").read().strip().splitlines()[-1])
print("parity", {k: d["parity"].get(k) for k in ("sentences", "identical", "identical_frac", "all_near_ties", "pass")})
print("cpu", json.dumps(d["cpu_baseline"])[:300]); print("clocks", d["clocks"], "hbm", d.get("peak_hbm_gb"), d.get("engine_device_gb"), d.get("engine_estimate_gb"))
r = json.loads(open("gpurun_out/bench_ref_final2.json").read().strip().splitlines()[-1]); print("ref", r["value"], r["cpu_baseline"]["kind"])
for l in open("gpurun_out/configs_final2.jsonl"):
    c = json.loads(l); print(c["config"]["workload"][:45], round(c["value"]), round(c["e2e"]["value"]))
PY
