for d in 0 8 16 24 2 26; do echo "== DBG=$d"; B=16 ONLY=gate_up DBG=$d timeout 30 python scratch/timeline.py 2>&1 | grep -E "mma issue|mma_end|deq0 lds|deq0 sttm|mma wait a_full|deq0 wait full"; done
