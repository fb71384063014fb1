timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
for e in "FNMT_LIVE_ROWS=0" "FNMT_LIVE_ROWS=1"; do env $e timeout 1200 python bench.py --model 6-6-8 --beam 4 --profile-sentences 0 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$e cfg4', d['value'])"; done
bash tools/gpu_ab.sh "FNMT_LIVE_ROWS=1"
