import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi+1:]
ki = h.index('Kernel Name'); mi = h.index('Metric Value'); ui = h.index('Metric Unit')
units = collections.Counter(r[ui] for r in data if len(r) > ui)
scale = {'nsecond':1e-3,'ns':1e-3,'usecond':1.0,'us':1.0,'msecond':1e3,'ms':1e3}
agg = collections.defaultdict(lambda: [0,0.0])
skip_prefix = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for r in data[skip_prefix:]:
    if len(r) <= mi: continue
    name = r[ki].replace('(anonymous namespace)::','')
    name = re.sub(r'^void ', '', name)
    name = name.split('(')[0]
    v = float(r[mi].replace(',','')) * scale.get(r[ui], 1.0)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v for _,v in agg.values())
print('units', dict(units), 'launches', sum(c for c,_ in agg.values()), 'total ms', round(tot/1e3,2))
for k,(c,v) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[3]) if len(sys.argv)>3 else 30]:
    print(f"{k[:70]:70s} {c:6d} {v/1e3:9.3f}ms {100*v/tot:5.1f}%")
