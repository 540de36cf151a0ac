for d in 0 2 4 8 16 6 14 30; do echo "== DEBUG=$d"; RTNQ_WGEMM_DEBUG=$d B=16 ONLY=o,gate_up python scratch/prof_layer.py; done > gpurun_out/variants.log 2>&1
B=16 python scratch/timeline.py > gpurun_out/timeline.log 2>&1
B=16 DBG=2 python scratch/timeline.py >> gpurun_out/timeline.log 2>&1
