mkdir -p gpurun_out
python tools/step_live.py 3072 20
python tools/step_live.py 1536 40
FNMT_GEMM_SMALLM=2 python tools/step_live.py 3072 20
FNMT_SPLITK=4 python tools/step_live.py 3072 20
