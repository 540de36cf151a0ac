# quick W4/W8 ffn_up + step numbers (bench.py --headline-only)
for b in ${BITS:-4}; do
python bench.py --headline-only --no-cpu-baseline --bits $b --steps 20 --sweep ${SWEEP:-1,16} > gpurun_out/q$b.json 2>gpurun_out/q$b.err || tail -3 gpurun_out/q$b.err
python -c "
import json; d=json.load(open('gpurun_out/q$b.json'))
print('W$b step', d['value'], 'ffn_up', d['roofline']['achieved'], d['roofline']['frac'], d['details']['sweep_gbs_by_batch'], 'layer us', d['details']['decode_layer_us'])"
done
