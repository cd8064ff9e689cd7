import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0]); tot=0
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',',''))
    v={'nsecond':1e-3,'ns':1e-3,'usecond':1,'us':1,'msecond':1e3,'ms':1e3}[r[ui]]*v
    agg[r[ki][:80]][0]+=1; agg[r[ki][:80]][1]+=v; tot+=v
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:20]:
    print(f"{t/1000:8.3f} ms {n:5d}  {k}")
print("total ms", tot/1000)
