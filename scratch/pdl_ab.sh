
RTNQ_DECODE_PDL=1 timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for bits in 4 8; do
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
RTNQ_PDL_EARLY=$1 RTNQ_DECODE_PDL=$2 timeout 300 python bench.py --bits $bits --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('bits=$bits early=$1 dpdl=$2', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'e2e', d['e2e']['value'], 'roof', d['roofline']['achieved'])"
done; done
