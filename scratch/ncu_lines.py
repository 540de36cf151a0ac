"""Executed warp instructions per CUDA source line of one kernel (ncu source page)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', 'regex:' + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, lines = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
    elif r and r[0] == 'Line No':
        hdr = r
    elif hdr and r and r[0].isdigit():
        ins = int(r[7]) if r[7].isdigit() else 0
        lines.append((ins, fname, int(r[0]), r[1][:120]))
tot = sum(l[0] for l in lines)
print(f"total executed warp instructions {tot}")
for ins, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * ins / tot:5.1f}% {ins:9d} {f}:{ln:<5d} {src}")
