# per-linear timings: current tcgen05 kernel vs the mma.sync v4 kernel (abc7d45)
for b in 1 4 16; do echo "== tc B=$b"; B=$b python scratch/prof_layer.py; done
for b in 1 4 16; do echo "== v4 B=$b"; PKGROOT=scratch/oldv4 B=$b python scratch/prof_layer.py; done
