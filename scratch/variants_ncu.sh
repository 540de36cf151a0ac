for b in 1 16; do for d in 0 1 2 3; do
  RTNQ_WGEMM_DEBUG=$d B=$b REPS=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wgemm --csv --log-file gpurun_out/ncu_v_b${b}_d${d}.csv python scratch/prof_layer.py > /dev/null 2>&1
done; done
