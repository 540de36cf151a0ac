for d in 0 64 128 2; do echo "== DBG=$d"; B=16 DBG=$d python scratch/timeline.py 2>&1 | grep -A18 gate_up | grep -E "gate_up|prod total|deq0 total|mma total|epi0 total|deq0 wait full"; done
