# A/B bench runs of the env switches given as arguments (each "NAME=VAL ..." string is one arm)
mkdir -p gpurun_out
for arm in "$@"; do
  echo "== arm: $arm"
  env $arm python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-sentences 0 > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", round(d["e2e"]["value"]), "ms/step", d["ms_per_step"], "clk", d["clocks"]["sm_mhz"])
PY
done
