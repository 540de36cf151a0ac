run() { env $2 timeout 300 python bench.py --bits $1 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('bits=$1 $2', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'roof', d['roofline']['achieved'])"; }
run 4 X=0; run 4 RTNQ_DECODE_PDL=1; run 8 X=0; run 8 RTNQ_DECODE_PDL=1; run 8 RTNQ_I8_PF=0; run 8 RTNQ_I8_PF=4
