mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_w4.json 2> gpurun_out/final/bench_w4.err
timeout 600 python bench.py --bits 8 > gpurun_out/final/bench_w8.json 2> gpurun_out/final/bench_w8.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
