# ffn_up / step for each library variant: LIBS="s84 s112 ..." BITS=4 bash scratch/ab_run.sh
for v in base $LIBS; do
  if [ $v = base ]; then export RTNQ_LIB=; else export RTNQ_LIB=paper_2505_15909_b200/librtnq_b200_$v.so; fi
  python bench.py --headline-only --no-cpu-baseline --bits ${BITS:-4} --steps 20 --sweep ${SWEEP:-1,16} > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', 'W${BITS:-4} step', d['value'], 'ffn_up', d['roofline']['achieved'], d['roofline']['frac'], d['details']['sweep_gbs_by_batch'])"
done
