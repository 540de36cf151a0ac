"""Summarise an ncu source page: top stalled SASS lines with context and per-barrier waits."""
import csv, sys, re, subprocess, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
out = []; h = None; seen = False
for r in rows:
    if r and r[0] == "Kernel Name":
        if seen: break
        seen = True; continue
    if r and r[0] == "Address": h = r; continue
    if h and len(r) == len(h): out.append(dict(zip(h, r)))
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(d[S]) for d in out)
print("samples", tot)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter()
for d in out:
    for c in cols: agg[c] += int(d[c] or 0)
print([(k, round(v / tot * 100, 1)) for k, v in agg.most_common(8)])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(range(len(out)), key=lambda i: -int(out[i][S]))[:n]
for i in sorted(top):
    d = out[i]
    prev = out[i - 1]["Source"].strip()[:60] if i else ""
    print(f"{int(d[S]) / tot * 100:5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:70]:70s} | prev: {prev}")
