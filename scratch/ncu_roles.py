"""Stall-reason samples of a kernel aggregated by source-line ranges (roles).
Usage: ncu_roles.py report kernel_regex file.cu name:lo-hi [name:lo-hi ...]"""
import csv, subprocess, sys
from collections import defaultdict
rep, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = [(a.split(':')[0], *map(int, a.split(':')[1].split('-'))) for a in sys.argv[4:]]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', 'regex:' + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, cur_line = None, None, None
agg = defaultdict(lambda: defaultdict(int))
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
    elif r and r[0] == 'Line No':
        hdr = r
    elif hdr and r and r[0].isdigit():
        cur_line = (fname, int(r[0]))
        d = dict(zip(hdr, r))
        role = 'other'
        if fname == src:
            for name, lo, hi in ranges:
                if lo <= cur_line[1] <= hi:
                    role = name
        elif fname and fname.endswith('.cuh'):
            role = 'helpers(' + fname + ')'
        for k_, v in d.items():
            if k_.startswith('stall_') and 'Not Issued' not in k_ and v.isdigit():
                agg[role][k_] += int(v)
        if r[4].isdigit():
            agg[role]['_samples'] += int(r[4])
        if r[7].isdigit():
            agg[role]['_instr'] += int(r[7])
tot = sum(a['_samples'] for a in agg.values())
for role, a in sorted(agg.items(), key=lambda x: -x[1]['_samples']):
    top = sorted(((v, k_) for k_, v in a.items() if k_.startswith('stall_')), reverse=True)[:6]
    print(f"{role:28s} samples {100 * a['_samples'] / max(tot, 1):5.1f}%  instr {a['_instr']:10d}  " +
          "  ".join(f"{k_[6:]}={100 * v / max(a['_samples'], 1):.0f}%" for v, k_ in top))
