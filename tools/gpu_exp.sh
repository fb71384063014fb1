run() { timeout 900 python bench.py --model 6-6-8 --beam 4 --chunk-sentences 8192 --profile-sentences 0 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('cfg4', d['value'])"; 
bash tools/gpu_ab.sh "FNMT_LANES=4" | tail -1; }
echo "hint 1ms"; run
make -C paper_2109_08003_b200/csrc clean > /dev/null; make -C paper_2109_08003_b200/csrc -j16 EXTRA=-DFNMT_MBAR_HINT_NS=0 > /dev/null 2>&1; echo "no hint"; run
make -C paper_2109_08003_b200/csrc clean > /dev/null; make -C paper_2109_08003_b200/csrc -j16 EXTRA=-DFNMT_MBAR_HINT_NS=20000 > /dev/null 2>&1; echo "hint 20us"; run
