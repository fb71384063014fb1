# norm-prefetch A/B + a --set full capture of the vocab argmax GEMM
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "norm or corpus or greedy" > gpurun_out/t_nm.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_nm.log
timeout 900 python bench.py > gpurun_out/bench_nm.json 2> gpurun_out/bench_nm.err; echo "bench rc=$?"
python tools/bsum.py gpurun_out/bench_nm.json
FNMT_LANES=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:gemm_tc_kernel<256, 4, 0, 0, 1, 2, 0>" --launch-skip 300 --launch-count 2 -o gpurun_out/full_r2v_vocab \
  python tools/profile_traffic.py r2v_vocab > gpurun_out/ncu_full_r2v_vocab.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full_r2v_vocab.log
