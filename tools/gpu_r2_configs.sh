# BASELINE configs 3-5 on the current kernels (builder-run lines)
mkdir -p gpurun_out
timeout 900 python bench.py --model 6-1-8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo "cfg3 rc=$?"
timeout 1200 python bench.py --model 6-6-8 --beam 4 --chunk-sentences 8192 --profile-sentences 2048 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
timeout 1200 python bench.py --model deep-12-768 --beam 4 --dtype bf16 --chunk-sentences 8192 --profile-sentences 2048 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; echo "cfg5 rc=$?"
cat gpurun_out/cfg3.json gpurun_out/cfg4.json gpurun_out/cfg5.json > gpurun_out/r02_configs.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/r02_configs.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"][:50], round(d["value"]), round(d["e2e"]["value"]), json.dumps(d.get("roofline"))[:200])
    for k, v in (d.get("kernel_profile") or {}).items(): print("   ", k, v)
PY
