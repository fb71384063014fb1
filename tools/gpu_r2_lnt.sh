for env in "FNMT_LAYER_KEYS=7" "FNMT_LAYER_KEYS=4" "FNMT_LAYER_KEYS=3" "FNMT_LAYER_KEYS=5" "FNMT_LAYER_KEYS=4 FNMT_LAYER_RING=3" "FNMT_LAYER_KEYS=3 FNMT_LAYER_RING=3" "FNMT_LAYER_KEYS=2 FNMT_LAYER_RING=4" "FNMT_LAYER_KEYS=6 FNMT_LAYER_RING=3"; do
  echo "== $env"; env $env python tools/step_live.py 3072 20 | sed -n 2p; env $env python tools/step_live.py 1536 40 | sed -n 2p; env $env python tools/step_live.py 768 80 | sed -n 2p
done
