import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
tot = collections.defaultdict(list)
unit = set()
for r in rows[hdr_i+1:]:
    name = r[ki].split('(')[0].replace('void csb::','').replace('csb::','')
    v = float(r[vi].replace(',',''))
    u = r[ui]; unit.add(u)
    v = v * {'nsecond':1e-3,'usecond':1,'msecond':1e3,'second':1e6}.get(u,1)
    tot[name].append(v)
allt = sum(sum(v) for v in tot.values())
print('units', unit)
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:32s} n={len(v):3d} mean={sum(v)/len(v):9.1f}us min={min(v):9.1f} max={max(v):9.1f} share={100*sum(v)/allt:5.1f}%")
