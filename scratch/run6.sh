for d in 0 2 4 8 16 6 30; do echo "== DBG=$d"; RTNQ_WGEMM_DEBUG=$d B=16 ONLY=gate_up,o timeout 60 python scratch/prof_layer.py | head -2; done
