# Round-2 full check: every GPU test, the default bench, the reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -q -m gpu -rs -s > gpurun_out/t_all.log 2>&1; echo "all rc=$?"
grep -E "parity:|near|passed|failed|FAILED|Error" gpurun_out/t_all.log | cut -c1-400 | tail -60
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
head -c 7000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
