for d in 0 512 258 770; do echo "== DBG=$d"; B=16 ONLY=gate_up DBG=$d timeout 60 python scratch/timeline.py | grep -E "deq_end|mma_end|epi_seg|mma total|mma wait|mma issue"; done
