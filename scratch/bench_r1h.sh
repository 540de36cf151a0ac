timeout 600 python bench.py > gpurun_out/r1h_bench_w4_b16.json 2> gpurun_out/r1h_bench_w4.err
timeout 600 python bench.py --bits 8 > gpurun_out/r1h_bench_w8_b16.json 2> gpurun_out/r1h_bench_w8.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1h_smoke.log 2>&1
