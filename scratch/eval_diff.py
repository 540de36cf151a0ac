"""Max relative difference of the GPU eval sweeps vs the reference's golden CSV."""
import csv, io, os, sys
sys.path.insert(0, os.getcwd())
from paper_2505_15909_b200 import eval as ev
cfg = ev.ToyConfig()
model = ev.FloatModel(cfg)
inputs = [ev.toy_input(cfg, i) for i in range(2)]
rows = []
for kind in ("first", "middle", "last"):
    rows += ev.horizontal_sweep(model, kind, inputs)
rows += ev.vertical_sweep(model, inputs)
got = list(csv.DictReader(io.StringIO(ev.sweep_to_csv(rows))))
want = list(csv.DictReader(open("tests/golden/toy_sweeps.csv")))
same = sum(g == w for g, w in zip(got, want))
mx = max(abs(float(g[k]) - float(w[k])) / max(abs(float(w[k])), 1e-300)
         for g, w in zip(got, want) for k in ("max_logit_dev", "mean_kl") if float(w[k]) != 0)
print(f"rows {len(got)}, CSV rows identical to the reference: {same}, max rel diff {mx:.3g}")
