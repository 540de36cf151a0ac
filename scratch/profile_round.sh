# Round evidence: bench line (N=1), ncu launch list of the bench command, one full ncu capture
set -x
mkdir -p gpurun_out/r1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r1/smi.txt
# warm clocks
timeout 60 python -c "import torch; a=torch.randn(8192,8192,device='cuda'); [a@a for _ in range(200)]; torch.cuda.synchronize()"
timeout 400 python bench.py > gpurun_out/r1/bench_w4.json 2> gpurun_out/r1/bench_w4.err
timeout 300 python bench.py --bits 8 --batch 16 --sweep 1,16,64 --no-cpu-baseline > gpurun_out/r1/bench_w8.json 2> gpurun_out/r1/bench_w8.err
timeout 300 python bench.py --impl reference > gpurun_out/r1/bench_ref.json 2> gpurun_out/r1/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wgemm -c 256 --csv --log-file gpurun_out/r1/launches_w4.csv python bench.py --steps 1 --warmup 3 --sweep 16 --no-cpu-baseline > gpurun_out/r1/ncu_bench.log 2>&1
B=16 NOTIME=1 NCOPY=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:wgemm -s 5 -c 4 -o gpurun_out/r1/full_w4_b16 python scratch/prof_layer.py > gpurun_out/r1/ncu_full.log 2>&1
