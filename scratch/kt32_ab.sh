run() { timeout 300 python $1 --bits 4 --steps 20 --sweep 16,32,64 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$2', c['sweep_gbs_by_batch'])"; }
run bench.py kt4_all; (cd scratch/basepkg && run bench.py base)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "w4 or chained or tensor_core" 2>&1 | tail -1
