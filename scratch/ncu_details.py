"""Print the key ncu --set full numbers of every kernel in a report (ncu -i ... --page details)."""
import csv, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2:] or ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy', 'Registers Per Thread',
        'Issue Slots Busy', 'No Eligible', 'Executed Instructions', 'Theoretical Occupancy', 'Warp Cycles Per Issued Instruction']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if any(d['Metric Name'] == w for w in want):
        print(d['ID'], d['Kernel Name'][:28], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
