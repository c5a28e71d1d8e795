import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    if d['Metric Name']!='gpu__time_duration.sum': continue
    k=d['Kernel Name'].split('(')[0].replace('void ','')[:40]
    v=float(d['Metric Value'].replace(',',''))
    u=d['Metric Unit']; v*= {'ns':1e-3,'nsecond':1e-3,'us':1,'usecond':1,'ms':1e3,'msecond':1e3}.get(u,1)
    agg[k][0]+=1; agg[k][1]+=v
tot=sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{k:40s} {v[0]:8d} {v[1]:10.1f} {v[1]/v[0]:8.1f} {v[1]/tot:6.3f}")
