mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -m pytest tests/test_gpu_corpus_parity.py tests/test_gpu_random_models.py -x -q -s -m gpu > gpurun_out/t_new.log 2>&1; echo "new rc=$?"
tail -30 gpurun_out/t_new.log
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_corpus_parity.py --deselect tests/test_gpu_random_models.py > gpurun_out/t_all.log 2>&1; echo "all rc=$?"
tail -15 gpurun_out/t_all.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
cat gpurun_out/bench1.json | head -c 6000; tail -5 gpurun_out/bench1.err
