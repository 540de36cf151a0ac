for pf in 0 2 4 8 0; do
RTNQ_I8_PF=$pf timeout 300 python bench.py --bits 8 --steps 30 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('pf=$pf', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'roof', d['roofline']['achieved'])"
done
