for d in 1024 3072 5120 9216 17408 31744; do echo "== DBG=$d"; B=16 ONLY=gate_up DBG=$d timeout 30 python scratch/timeline.py 2>&1 | grep -E "isolated|Error"; done
