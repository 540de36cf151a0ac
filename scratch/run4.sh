timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for b in 1 16; do B=$b python scratch/prof_layer.py; done 2>&1
for b in 1 16 64; do BITS=8 B=$b python scratch/prof_layer.py; done 2>&1
B=16 python scratch/timeline.py 2>&1 | grep -A22 gate_up
B=1 python scratch/timeline.py 2>&1 | grep -A22 gate_up
