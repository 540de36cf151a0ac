"""Opcode histogram (executed warp instructions) of one kernel in an ncu report."""
import csv, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(h) - 2 and r[0].startswith('0x')]
iE, iS = h.index('Instructions Executed'), h.index('Source')
tot = sum(int(r[iE] or 0) for r in data)
print('total warp instr', tot, 'sass lines', len(data))
c = Counter()
for r in data:
    t = r[iS].split()
    if not t:
        continue
    op = t[1] if t[0].startswith('@') else t[0]
    c[op.split('.')[0] if len(sys.argv) < 4 else op] += int(r[iE] or 0)
for op, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{op:24s} {v:12d} {100 * v / tot:5.1f}")
