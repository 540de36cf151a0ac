RTNQ_WGEMM_DEBUG=2 B=16 NOTIME=1 REPS=1 ncu --set full --import-source on --clock-control none -k regex:wgemm -s 1 -c 1 -o gpurun_out/prof_o_conly python scratch/prof_layer.py > /dev/null 2>&1
for c in 16 64 148 296; do
RTNQ_WGEMM_CTAS=$c RTNQ_WGEMM_DEBUG=2 B=16 NOTIME=1 REPS=2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgemm --csv --log-file gpurun_out/ncu_conly_ctas$c.csv python scratch/prof_layer.py > /dev/null 2>&1
done
