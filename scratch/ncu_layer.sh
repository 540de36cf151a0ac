# kernel durations (ncu) for one layer at B=1/16, W4; plus the bench graph
for b in 1 16; do
  B=$b REPS=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:wgemm --csv --log-file gpurun_out/ncu_l_b${b}.csv python scratch/prof_layer.py > /dev/null 2>&1
done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w4.log 2>&1
