timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for b in 1 16; do B=$b python scratch/prof_layer.py; done > gpurun_out/prof.log 2>&1
for b in 1 16 64; do BITS=8 B=$b python scratch/prof_layer.py; done >> gpurun_out/prof.log 2>&1
B=16 python scratch/timeline.py > gpurun_out/tl.log 2>&1
