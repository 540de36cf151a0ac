import csv, glob, sys
for f in sorted(glob.glob(sys.argv[1])):
    rows=list(csv.reader(open(f)))
    st=None
    for i,r in enumerate(rows):
        if 'Metric Value' in r: h=r; st=i+1; break
    if st is None: print(f, 'no data'); continue
    vals={}
    for r in rows[st:]:
        d=dict(zip(h,r)); vals.setdefault(d['ID'],{})[d['Metric Name']]=float(d['Metric Value'].replace(',',''))
    out=[]
    for k in sorted(vals,key=int)[-4:]:
        t=vals[k]['gpu__time_duration.sum']; b=vals[k]['dram__bytes_read.sum']
        out.append(f"{t/1000:6.1f}us/{b/t:5.0f}GB/s")
    print(f.split('/')[-1], ' '.join(out))
