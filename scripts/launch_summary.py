import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
H=rows[h]; ki=H.index("Kernel Name"); vi=H.index("Metric Value")
d=collections.defaultdict(list)
for r in rows[h+1:]:
    d[r[ki][:70]].append(float(r[vi])/1e3)
for k,v in d.items(): print(f"{len(v):3d} {sum(v)/len(v):9.2f} us  {k}")
