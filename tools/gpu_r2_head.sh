# Round-2 re-entry check of HEAD: every GPU test, smoke, the default bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1800 python -m pytest tests -q -m gpu -rs -s > gpurun_out/t_${TAG:-head}.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/t_${TAG:-head}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-head}.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG:-head}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG:-head}.json 2> gpurun_out/bench_${TAG:-head}.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_${TAG:-head}.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "roofline", json.dumps(d["roofline"]))
print("parity", {k: d["parity"].get(k) for k in ("sentences", "identical", "identical_frac", "all_near_ties", "pass")})
print("clocks", d["clocks"])
for k, v in d["kernel_profile"].items(): print(k, v)
PY
