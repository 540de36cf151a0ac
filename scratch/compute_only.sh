for b in 1 16; do
  B=$b NOTIME=1 REPS=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wgemm --csv --log-file gpurun_out/ncu_full_b${b}.csv python scratch/prof_layer.py > /dev/null 2>&1
  RTNQ_WGEMM_DEBUG=2 B=$b NOTIME=1 REPS=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wgemm --csv --log-file gpurun_out/ncu_conly_b${b}.csv python scratch/prof_layer.py > /dev/null 2>&1
done
