run() { timeout 300 python $1 --bits 4 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$2', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'roof', d['roofline']['achieved'])"; }
run bench.py kt4_16; (cd scratch/basepkg && run bench.py base); run bench.py kt4_16
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "w4 or chained or llama or 405b or cluster or tensor_core" 2>&1 | tail -1
