import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    if d['Metric Name']!='gpu__time_duration.sum': continue
    name=d['Kernel Name'][:90]
    v=float(d['Metric Value'].replace(',',''))
    u=d['Metric Unit']
    v = v/1e3 if u=='nsecond' or u=='ns' else (v*1e3 if u in('msecond','ms') else v)  # -> us
    agg[name][0]+=1; agg[name][1]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}% n={v[0]:5d} avg {v[1]/v[0]:9.1f}us  {k}")
print("total ms", tot/1e3, "launches", sum(v[0] for v in agg.values()))
