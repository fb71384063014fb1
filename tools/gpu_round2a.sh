mkdir -p gpurun_out
python -m pytest tests/test_gpu_corpus_parity.py -q -x -s -m gpu -k "greedy or logits" > gpurun_out/t_corpus.log 2>&1; echo "corpus rc=$?"
grep -E "parity:|rel err|passed|failed" gpurun_out/t_corpus.log | cut -c1-400
python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/t_all.log
bash tools/gpu_ab.sh "FNMT_DEC_BULK=0" "FNMT_DEC_BULK=1" "FNMT_DEC_BULK=0" "FNMT_DEC_BULK=1"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench2.json').read().strip().splitlines()[-1])
for k in ('value','e2e','roofline','parity','cpu_baseline'): print(k, json.dumps(d.get(k))[:1500])
print(json.dumps(d.get('kernel_profile')))"
