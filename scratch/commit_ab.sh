run() { timeout 300 python $1 --bits $3 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$2 w$3', d['value'], c['sweep_gbs_by_batch'], 'layer_us', c['decode_layer_us'], 'roof', d['roofline']['achieved'])"; }
for b in 4 8; do run bench.py leader_commits $b; (cd scratch/basepkg && run bench.py base $b); done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
