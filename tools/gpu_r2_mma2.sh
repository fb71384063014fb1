for st in 2 3; do FNMT_LAYER_STAGES=$st python tools/step_live.py 3072 20 | head -3; done
FNMT_LAYER_STAGES=2 python tools/step_live.py 1536 40 | head -3
FNMT_LAYER_MMA=0 python tools/step_live.py 1536 40 | head -3
