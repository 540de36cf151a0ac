timeout 60 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 || exit 1
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for b in 1 16; do B=$b timeout 60 python scratch/prof_layer.py; done 2>&1
for b in 1 16 64; do BITS=8 B=$b timeout 60 python scratch/prof_layer.py; done 2>&1
B=16 timeout 60 python scratch/timeline.py 2>&1 | grep -A24 "^gate_up"
