for d in 0 131072 262144 393216; do echo "== DBG=$d"; RTNQ_WGEMM_DEBUG=$d B=16 ONLY=gate_up,o timeout 30 python scratch/prof_layer.py | head -2; done
