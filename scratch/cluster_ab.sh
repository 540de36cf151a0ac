for bits in 8 4; do
for cl in 1 0; do
RTNQ_WGEMM_CLUSTER=$cl timeout 300 python bench.py --bits $bits --steps 30 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('bits=$bits cluster=$cl', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'roof', d['roofline']['achieved'])"
done; done
