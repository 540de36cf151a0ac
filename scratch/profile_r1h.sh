#!/bin/bash
# Round-1 (second session) profile pass: bench lines, ncu launch lists, one full capture.
set -x
mkdir -p gpurun_out/r1h
timeout 300 python -m pytest tests -m gpu -q > gpurun_out/r1h/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h/smoke.log 2>&1
for b in 4 8; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r1h/launches_w${b}.csv python bench.py --bits $b --steps 1 --warmup 3 --layers 2 --sweep 16 --no-cpu-baseline > /dev/null 2>&1
done
BITS=4 B=16 ONLY=gate_up NOTIME=1 REPS=2 NCOPY=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgemm_i4 -s 1 -c 1 \
  -o gpurun_out/r1h/i4_gate_up_b16 python scratch/prof_layer.py > /dev/null 2>&1
BITS=8 B=16 ONLY=gate_up NOTIME=1 REPS=2 NCOPY=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgemm_i8 -s 1 -c 1 \
  -o gpurun_out/r1h/i8_gate_up_b16 python scratch/prof_layer.py > /dev/null 2>&1
ls -la gpurun_out/r1h
