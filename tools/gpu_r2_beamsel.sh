# beam select: lane-parallel candidate loads — beam tests, config 4 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "beam" > gpurun_out/t_bs.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_bs.log
timeout 1500 python bench.py --model 6-6-8 --beam 4 --profile-sentences 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bs_cfg4.json 2> gpurun_out/bs_cfg4.err; echo "cfg4 rc=$?"
python tools/bsum.py gpurun_out/bs_cfg4.json
