timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for d in 0 1 0 1; do
RTNQ_I8_DIRECT=$d timeout 300 python bench.py --bits 8 --steps 30 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('direct=$d', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'e2e', d['e2e']['value'], 'roof', d['roofline']['achieved'])"
done
